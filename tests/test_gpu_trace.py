"""K6 (gsb_trace_parse / gsb_trace_format) on the GPU vs the restated load_trace /
save_trace_csv (oracle/gs_trace.c, pinned to the reference by tests/test_oracle_trace.py) and
the reference's own results committed in tests/golden/trace_cases.json."""
import json
import os

import numpy as np
import pytest
import torch

from trace_cases import CASES, H3, H4, tile_straddle_case

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "trace_cases.json")


def _gpu(eng, data, thr):
    from paper_2508_16449_b200 import api
    try:
        t = eng.parse_trace(data, thr)
    except api.TraceError as e:
        return {"error": [e.kind, e.row, str(e)]}
    return {"arrival": t.arrival_ms.cpu().tolist(), "prompt": t.prompt_tokens.cpu().tolist(),
            "output": t.output_tokens.cpu().tolist(), "cls": t.slo_class.cpu().tolist()}


def _norm(r):
    if isinstance(r[0], str):
        return {"error": [r[1], r[2], r[3]]}
    return {"arrival": [int(x) for x in r[0]], "prompt": [int(x) for x in r[1]],
            "output": [int(x) for x in r[2]], "cls": [int(x) for x in r[3]]}


@pytest.mark.parametrize("name,data,thr", CASES, ids=[c[0] for c in CASES])
def test_parse_fixture_equals_reference(gsb, restate, name, data, thr):
    gold = json.load(open(GOLD))[name]
    got = _gpu(gsb, data, thr)
    assert got == gold
    assert got == _norm(restate.trace_parse(data, thr))


@pytest.mark.parametrize("crlf", [False, True])
def test_parse_tile_straddling_file(gsb, restate, crlf):
    data = tile_straddle_case(20000, crlf)  # ~0.4 MB: lines across 4 KB tiles, long lines
    assert _gpu(gsb, data, 1024) == _norm(restate.trace_parse(data, 1024))


def _day_trace(restate, cls=True):
    a, p, o = restate.gen_poisson_trace(5.0, 86_400_000, seed=12)  # Azure-day scale, 432k rows
    c = (p > 1024).astype(np.uint8)
    return a, p, o, c, restate.trace_format(a, p, o, c if cls else None)


def test_parse_day_trace_bit_exact(gsb, restate):
    a, p, o, c, text = _day_trace(restate)
    t = gsb.parse_trace(text, 1024, name="day")
    assert t.has_class_column
    assert torch.equal(t.arrival_ms.cpu(), torch.from_numpy(a))
    assert torch.equal(t.prompt_tokens.cpu(), torch.from_numpy(p))
    assert torch.equal(t.output_tokens.cpu(), torch.from_numpy(o))
    assert torch.equal(t.slo_class.cpu(), torch.from_numpy(c))
    assert t.duration_ms == int(a[-1]) and t.nominal_qps == 1000.0 * len(a) / int(a[-1])


@pytest.mark.parametrize("kind", ["bad_field", "non_monotone", "two_errors", "mismatch"])
def test_error_deep_in_large_file(gsb, restate, kind):
    a, p, o, c, text = _day_trace(restate)
    lines = text.split(b"\n")
    k = 300_001  # a row near the end (line index k, row counter k + 1)
    if kind == "bad_field":
        lines[k] = lines[k].replace(b",", b",x", 1)
    elif kind == "non_monotone":
        f = lines[k].split(b",")
        f[0] = b"%d" % (int(a[k - 2]) - 1)
        lines[k] = b",".join(f)
    elif kind == "two_errors":
        lines[k + 5000] = b"1,2"
        lines[k] = lines[k] + b",extra"
    else:
        f = lines[k].split(b",")
        f[3] = b"L" if f[3] == b"SM" else b"SM"
        lines[k] = b",".join(f)
    bad = b"\n".join(lines)
    got = _gpu(gsb, bad, 1024)
    assert got == _norm(restate.trace_parse(bad, 1024))
    assert got["error"][1] == k + 1


def test_parse_from_device_bytes_and_file(gsb, restate, tmp_path):
    data = tile_straddle_case(3000)
    dev = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    assert _gpu(gsb, dev, 1024) == _norm(restate.trace_parse(data, 1024))
    f = tmp_path / "azure.csv"
    f.write_bytes(data)
    t = gsb.load_trace(str(f), 1024)
    assert t.name == "azure"
    from paper_2508_16449_b200 import api
    with pytest.raises(api.TraceError, match="cannot open trace file"):
        gsb.load_trace(str(tmp_path / "missing.csv"))


def test_format_equals_restated_writer(gsb, restate):
    rng = np.random.default_rng(9)
    n = 100_000
    a = np.sort(rng.integers(0, 10**13, n)).astype(np.int64)
    a[:4] = [-5, np.iinfo(np.int64).min, np.iinfo(np.int64).max, 0]
    p = rng.integers(-(2**31), 2**31 - 1, n, dtype=np.int64).astype(np.int32)
    p[:2] = [np.iinfo(np.int32).min, np.iinfo(np.int32).max]
    o = rng.integers(1, 5000, n).astype(np.int32)
    c = (p > 1024).astype(np.uint8)
    for cls in (None, c):
        assert gsb.format_trace(a, p, o, cls) == restate.trace_format(a, p, o, cls)
    assert gsb.format_trace(a[:0], p[:0], o[:0], c[:0]) == H4 + b"\n"
    assert gsb.format_trace(a[:0], p[:0], o[:0]) == H4 + b"\n"  # all_of over nothing
    assert gsb.format_trace(a[:1], p[:1], o[:1]) == H3 + b"\n" + restate.trace_format(
        a[:1], p[:1], o[:1]).split(b"\n", 1)[1]


def test_round_trip_and_route(gsb, restate, tmp_path):
    """CSV on disk -> K6 -> K1 on the device-resident SoA, never leaving the GPU."""
    from paper_2508_16449_b200 import api
    a, p, o, c, text = _day_trace(restate)
    f = tmp_path / "day.csv"
    f.write_bytes(text)
    t = gsb.load_trace(str(f))
    gsb.save_trace_csv(t, str(tmp_path / "back.csv"))
    assert (tmp_path / "back.csv").read_bytes() == text
    gsb.set_profiles([api.GpuProfile.default_profile()])
    rr_csv = gsb.route_bin(t.arrival_ms, t.prompt_tokens, api.RoutingConfig(True, [512, 1024],
                                                                          [0, 1, 2]), 60_000)
    rr_np = gsb.route_bin(a, p, api.RoutingConfig(True, [512, 1024], [0, 1, 2]), 60_000)
    assert torch.equal(rr_csv.cls, rr_np.cls) and torch.equal(rr_csv.count, rr_np.count)
    assert torch.equal(rr_csv.t_ref.view(torch.int64), rr_np.t_ref.view(torch.int64))


def test_graph_survives_scratch_growth(gsb, restate):
    """A CUDA graph captured over the fused K2 (which uses the context's scratch) stays valid
    after a later call grows the scratch (a large trace parse): outgrown scratch buffers are
    retired, not freed, so the graph's addresses remain live."""
    from paper_2508_16449_b200 import api
    gsb.set_profiles([api.GpuProfile.default_profile()])
    a, p, _ = restate.gen_poisson_trace(5.0, 3_600_000, seed=8)
    d_a = torch.as_tensor(a, device="cuda")
    d_p = torch.as_tensor(p, device="cuda")
    routing = api.RoutingConfig(True, [512, 1024], [0, 1, 2])
    rr = gsb.route_bin(d_a, d_p, routing, 60_000)
    summ = gsb.summary_buffer(3)
    sel = gsb.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=57_000.0, summary_out=summ)
    want_f, want_s = sel.f_idx.clone(), summ.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            gsb.route_bin(d_a, d_p, routing, 60_000, 0, rr.n_windows, out=rr)  # no host reads
            gsb.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=57_000.0, out=sel,
                               summary_out=summ)
    torch.cuda.current_stream().wait_stream(s)
    _, _, _, _, text = _day_trace(restate)
    gsb.parse_trace(text)  # grows the scratch well past the graph's partial buffer
    sel.f_idx.zero_()
    summ.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(sel.f_idx, want_f)
    assert torch.equal(summ, want_s)


def test_cap_rows_overflow_is_reported_then_parses(gsb, restate):
    """gsb_trace_parse with cap_rows below the row count: INVALID_ARGUMENT with the true count
    (rows past the cap are never written: the buffers below are guarded), then the same bytes
    with room parse to the restated load_trace's rows; a bad header wins over the cap."""
    import ctypes as C
    from paper_2508_16449_b200 import _lib as L
    rng = np.random.default_rng(3)
    n = 5000
    a = np.cumsum(rng.integers(0, 5, n))
    lines = [H3.decode()] + [f"{a[i]},{rng.integers(1, 4000)},{rng.integers(1, 900)}"
                             for i in range(n)]
    data = ("\n".join(lines) + "\n").encode()
    dev = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()

    def call(cap, buf=None):
        guard = 64
        arr = torch.full((cap + guard,), -7, dtype=torch.int64, device="cuda")
        prm = torch.full((cap + guard,), -7, dtype=torch.int32, device="cuda")
        out = torch.full((cap + guard,), -7, dtype=torch.int32, device="cuda")
        cls = torch.full((cap + guard,), 7, dtype=torch.uint8, device="cuda")
        res = L.CTraceResult()
        b = dev if buf is None else buf
        rc = gsb.lib.gsb_trace_parse(gsb.ctx, C.c_void_p(b.data_ptr()), b.numel(), 1024, cap,
                                     C.c_void_p(arr.data_ptr()), C.c_void_p(prm.data_ptr()),
                                     C.c_void_p(out.data_ptr()), C.c_void_p(cls.data_ptr()),
                                     C.byref(res), None)
        torch.cuda.synchronize()
        return rc, res, arr, prm, out, cls

    rc, res, arr, prm, out, cls = call(1000)
    assert rc == L.INVALID_ARGUMENT and res.n_rows == n
    assert (arr[1000:] == -7).all() and (prm[1000:] == -7).all() and (cls[1000:] == 7).all()
    rc, res, arr, prm, out, cls = call(n)
    assert rc == L.OK and res.n_rows == n and res.max_arrival_ms == a[-1]
    want = restate.trace_parse(data, 1024)
    for got, w in zip((arr, prm, out, cls), want[:4]):
        np.testing.assert_array_equal(got[:n].cpu().numpy(), w)
    bad = torch.frombuffer(bytearray(b"arrival,prompt\n" + data[len(H3) + 1:]), dtype=torch.uint8).cuda()
    rc, res, *_ = call(10, bad)
    assert rc == L.TRACE_ERROR and L.TRACE_KINDS[res.kind] == "BadHeader" and res.row == 1
