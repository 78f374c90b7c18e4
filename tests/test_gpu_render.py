"""f4: the simulator's CSV wire formats rendered on the GPU (gsb_freq_timeline_csv,
gsb_prefill_commands_csv) against the unmodified reference's freq_timeline_csv /
prefill_commands_csv (simkernel.cpp:686-714, '%.10g' via snprintf), byte for byte: on the
decode pool's clock changes from K5 and on prefill commands from K2, plus a value sweep over the
%.10g edge cases (rounding ties, decade boundaries, %e switch-overs, subnormals, inf/nan)."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _edge_values(rng):
    v = [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1.5, 2.5, 0.0001, 0.00001, 1e-5, 9.9999999995e-5,
         123456789.0, 1234567890.0, 12345678901.0, 9999999999.0, 9999999999.5, 9999999998.5,
         99999.999995, 0.99999999995, 1e10, 1e9, 999999999.5, 1e21, 1e-300, 5e-324, 2.2250738585072014e-308,
         1.7976931348623157e308, math.inf, -math.inf, math.nan, 1410.0, 210.0, 25721.25,
         60000.0 * 123456, 0.95 * 57000.0, 1 / 3, 2 / 3, 1e100 / 3, 123.45678905, 123.45678915]
    v += list(rng.uniform(-1e6, 1e6, 300)) + list(10.0 ** rng.uniform(-30, 30, 300))
    # exact ties at the 10th significant digit: d.ddddddddd5 x 10^k with short binary forms
    v += [int(x) / 2 ** 4 for x in rng.integers(10 ** 10, 10 ** 12, 200)]
    v += list(np.round(rng.uniform(0, 1e6, 200), 3)) + list(rng.integers(0, 2 ** 40, 100) * 0.25)
    return np.array(v, np.float64)


def test_format_g10_matches_reference(gsb, ref):
    rng = np.random.default_rng(4)
    vals = _edge_values(rng)
    got = gsb.format_g10(vals)
    want = ref.freq_timeline_csv(vals, np.zeros(len(vals)), np.zeros(len(vals)),
                                 np.zeros(len(vals))).decode().splitlines()[1:]
    want = [w.split(",")[0] for w in want]
    bad = [(x, g, w) for x, g, w in zip(vals, got, want) if g != w]
    assert not bad, bad[:10]


def test_freq_timeline_csv_from_the_decode_pool(gsb, ref, restate):
    """K5's per-worker clock changes of a closed-loop scenario (d_freq: applied_ms, f), rendered
    as the simulator's timeline (decode pool) plus random prefill-pool records."""
    from paper_2508_16449_b200 import api, workloads as wl
    pa, pp, po = wl.sinusoid_decode_trace(1500.0, 1000.0, 120_000.0, 60_000, seed=11)
    stream = wl.decode_stream(pa, pp, po)
    cfgs = wl.pool_sweep(4)
    plan = gsb.decode_pool(cfgs, stream, api.GpuProfile.default_profile(), api.SimConfig(),
                           api.SloConfig(), freq_cap=4096, launch=False)
    plan["out"]["freq"].zero_()  # entries past each worker's changes stay (0, 0)
    gsb.run_pool(plan)
    torch.cuda.synchronize()
    fr = plan["out"]["freq"].cpu().numpy()      # [N][W][cap][2]
    assert fr.ndim == 4
    recs = fr[0].reshape(-1, 2)
    keep = recs[:, 0] > 0
    applied, f = recs[keep, 0], recs[keep, 1]
    worker = np.repeat(np.arange(fr.shape[1]), fr.shape[2])[keep]
    rng = np.random.default_rng(1)
    applied = np.concatenate([applied, rng.uniform(0, 1e7, 500)])
    f = np.concatenate([f, 210.0 + 15.0 * rng.integers(0, 81, 500)])
    worker = np.concatenate([worker, rng.integers(0, 8, 500)]).astype(np.int32)
    pool = np.concatenate([np.zeros(keep.sum(), np.uint8), np.ones(500, np.uint8)])
    got = gsb.freq_timeline_csv(applied, pool, worker, f)
    assert got == ref.freq_timeline_csv(applied, pool, worker, f)
    assert keep.sum() > 10


def test_prefill_commands_csv_from_k2(gsb, ref):
    """K2's commands of a DEADLINE_SLACK pass (per non-empty cell: window start, class, a
    worker, the chosen clock or f_max, the window, the infeasible flag)."""
    from paper_2508_16449_b200 import api, workloads as wl
    gsb.set_profiles([api.GpuProfile.default_profile()])
    a, p, _ = wl.poisson_trace(5.0, 300 * 60_000, "alibaba_chat", seed=2)
    routing = api.RoutingConfig(True, wl.THRESHOLDS[3], [0, 1, 2])
    rr = gsb.route_bin(a, p, routing, 60_000, 0, 300, want_deadline=True)
    cols = []
    for sel in (gsb.prefill_select(rr, api.L.DEADLINE_SLACK, qopt=api.QueueOptimizerConfig()),
                gsb.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=57_000.0)):
        torch.cuda.synchronize()
        fi = sel.f_idx.cpu().numpy()[0]
        live = np.flatnonzero(fi != -2)
        cols.append(((live // 3) * 60_000.0, (live % 3).astype(np.int32),
                     np.where(fi[live] >= 0, 210.0 + 15.0 * fi[live], 1410.0),
                     sel.window_ms.cpu().numpy()[live], (fi[live] < 0).astype(np.uint8)))
    tick, cls, f, win, inf = (np.concatenate(c) for c in zip(*cols))
    got = gsb.prefill_commands_csv(tick, cls, cls, f, win, inf)
    assert got == ref.prefill_commands_csv(tick, cls, cls, f, win, inf)
    assert inf.sum() > 0 and (inf == 0).sum() > 0
    assert gsb.prefill_commands_csv([], [], [], [], [], []) == ref.prefill_commands_csv(
        [], [], [], [], [], [])


def _edge_values6(rng):
    v = [0.0, -0.0, 1.0, 0.1, 1.5, 2.5, 1e-5, 0.0001, 0.000123456789, 9.999995e-5, 999999.0,
         999999.5, 9999995.0, 999999.4999, 1234565.0, 1234575.0, 123456.5, 123457.5, 1e6, 1e15,
         5e-324, 1.7976931348623157e308, math.inf, -math.inf, math.nan, 1410.0, 25.125, 0.95,
         60000.0 * 0.95, 1 / 3, 2 / 3, 123.4565, 100.0 / 7]
    v += list(rng.uniform(-1e6, 1e6, 300)) + list(10.0 ** rng.uniform(-30, 30, 300))
    # exact ties at the 6th significant digit: d.dddd5 x 10^k with short binary forms
    v += [int(x) / 2 ** 3 for x in rng.integers(10 ** 6, 10 ** 8, 300)]
    v += list(np.round(rng.uniform(0, 1e4, 300), 2))
    return np.array(v, np.float64)


def test_format_g6_matches_reference(gsb, ref):
    """'%.6g' (decode_ctl.cpp fmt_num) on the GPU against the reference's own decision_log_csv
    rendering the same values (tick_ms column)."""
    from paper_2508_16449_b200 import api
    rng = np.random.default_rng(6)
    vals = _edge_values6(rng)
    got = gsb.format_g(vals, 6)
    rec = np.zeros(len(vals), api.DECISION_DTYPE)
    rec["tick_ms"] = vals
    want = [w.split(",")[0] for w in ref.decision_log_csv(rec).decode().splitlines()[1:]]
    bad = [(x, g, w) for x, g, w in zip(vals, got, want) if g != w]
    assert not bad, bad[:10]


def test_decision_log_csv_from_the_decode_pool(gsb, ref):
    """K5's per-worker controller decision logs (every action kind), rendered on the GPU as the
    reference's decision_log_csv, byte for byte; plus random records over every field."""
    from paper_2508_16449_b200 import api, workloads as wl
    pa, pp, po = wl.sinusoid_decode_trace(1500.0, 1000.0, 120_000.0, 60_000, seed=11)
    stream = wl.decode_stream(pa, pp, po)
    cfgs = wl.pool_sweep(3)
    plan = gsb.decode_pool(cfgs, stream, api.GpuProfile.default_profile(), api.SimConfig(),
                           api.SloConfig(), rec_cap=6000, launch=False)
    plan["out"]["records"].zero_()
    gsb.run_pool(plan)
    torch.cuda.synchronize()
    rec = plan["out"]["records"].cpu().numpy().view(api.DECISION_DTYPE)[..., 0]  # [N][W][cap]
    r = rec[0].reshape(-1)
    r = r[r["tick_ms"] > 0]
    assert len(r) > 100 and len(set(r["action"].tolist())) >= 4
    assert gsb.decision_log_csv(r) == ref.decision_log_csv(r)
    # the device tensor path gives the same bytes
    dev = torch.from_numpy(r.view(np.uint8).copy()).cuda()
    assert gsb.decision_log_csv(dev) == ref.decision_log_csv(r)
    rng = np.random.default_rng(2)
    x = np.zeros(400, api.DECISION_DTYPE)
    for f in ("tick_ms", "tps", "p95_tbt_ms", "band_lo", "band_hi", "command_mhz"):
        x[f] = 10.0 ** rng.uniform(-6, 9, 400) * rng.choice([-1, 1], 400)
    x["worker"] = rng.integers(-5, 1 << 30, 400)
    x["bucket"] = rng.integers(-1, 40, 400)
    x["action"] = rng.integers(0, 8, 400)
    assert gsb.decision_log_csv(x) == ref.decision_log_csv(x)
    assert gsb.decision_log_csv(x[:0]) == ref.decision_log_csv(x[:0])
