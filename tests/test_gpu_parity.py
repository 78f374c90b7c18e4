"""GPU parity: the sm_100a kernels behind include/gsb.h against the CPU oracle
(oracle/gs_oracle.c) and the unmodified reference build (oracle/_ref). Bit-exact for every
integer output, chosen clock and energy; run with `pytest -m gpu` on a B200."""
import math

import numpy as np
import pytest
import torch

from oracle.oracle import (Profile, TelemetryArrays, band_table, default_ctl_cfg,
                           default_qopt_cfg)

pytestmark = pytest.mark.gpu

LEVELS = np.arange(200.0, 3000.0 + 1e-9, 200.0)


def u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _api():
    from paper_2508_16449_b200 import api
    return api


def synth_profiles(api):
    """default + 3 synthetic variants (synth-* profiles, validated)."""
    base = api.GpuProfile.default_profile()
    out = [base]
    for i, (ls, ps) in enumerate([(1.6, 1.25), (0.7, 0.8), (2.5, 1.6)]):
        p = api.GpuProfile(f"synth-{i}", base.grid,
                           api.LatencyModel(base.prefill.a * ls, base.prefill.b * ls,
                                            base.prefill.c * ls, 1410.0),
                           base.decode,
                           api.PowerModel(base.power.k3 * ps, base.power.k2 * ps,
                                          base.power.k1 * ps, base.power.k0 * ps,
                                          base.power.p_idle_w * ps))
        p.validate()
        out.append(p)
    return out


def to_oracle(p) -> Profile:
    return Profile(*p.key())


@pytest.fixture(scope="module")
def eng(gsb):
    return gsb


def test_library_is_native_and_on_b200(eng):
    name = torch.cuda.get_device_name(0)
    cap = torch.cuda.get_device_capability(0)
    assert cap[0] == 10, (name, cap)
    assert eng.lib.gsb_version().startswith(b"gsb")


def test_fast_division_equals_ieee(eng):
    """div_pre (precomputed reciprocal + 2 FMA) == IEEE division for every grid clock and
    1000, over random dividends across the exponent range and near-midpoint hard cases."""
    bad = eng.selftest_division(1 << 22)
    assert bad == 0


@pytest.mark.parametrize("thr,P,qps,wms", [
    ([512, 1024], 1, 5.0, 60_000),
    ([256, 512, 1024, 2048], 2, 3.0, 60_000),
    ([128, 256, 512, 768, 1024, 2048, 4096], 4, 8.0, 30_000),
    ([1024], 3, 20.0, 1_000),
    # windows far larger than one warp's staging chunk (kRouteCap): chains continue across chunks
    ([512, 1024], 4, 150.0, 60_000),
    ([256, 512, 1024, 2048], 1, 40.0, 30_000),
    # sparse: most windows empty, window edges far apart
    ([512, 1024, 4096], 2, 0.02, 1_000),
])
# want_deadline False selects the FIXED-mode K1b instances (k_route_bin<C, P, DL=0, G>), the ones
# the bench times; True the deadline instances
@pytest.mark.parametrize("want_deadline", [True, False])
def test_route_bin_matches_oracle(eng, restate, thr, P, qps, wms, want_deadline):
    api = _api()
    profs = synth_profiles(api)[:P]
    eng.set_profiles(profs)
    a, p, _ = restate.gen_poisson_trace(qps, 1_800_000, 768.0, 3072.0, 0.15, 128.0, seed=len(thr))
    nw = int(a[-1] // wms) + 1
    rr = eng.route_bin(a, p, api.RoutingConfig(True, thr, list(range(len(thr) + 1))), wms, 0, nw,
                       want_deadline=want_deadline, want_fifo=True)
    torch.cuda.synchronize()
    cls, cnt, tref, mdl, fifo = restate.route_bin(a, p, thr, wms, 0, nw,
                                                  [to_oracle(x) for x in profs])
    np.testing.assert_array_equal(rr.cls.cpu().numpy(), cls)
    np.testing.assert_array_equal(rr.count.cpu().numpy().view(np.uint32), cnt)
    np.testing.assert_array_equal(u64(rr.t_ref.cpu().numpy()), u64(tref))
    if want_deadline:
        np.testing.assert_array_equal(u64(rr.min_deadline.cpu().numpy()), u64(mdl))
    else:
        assert rr.min_deadline is None
    # the non-empty cell list K1b emits in the same pass (decoupled look-back across CTAs)
    n_ne = int(rr.n_nonempty.item())
    np.testing.assert_array_equal(rr.nonempty.cpu().numpy()[:n_ne].view(np.uint32),
                                  np.flatnonzero(cnt).astype(np.uint32))
    np.testing.assert_array_equal(rr.fifo.cpu().numpy(), fifo)
    eng.set_profiles([api.GpuProfile.default_profile()])


@pytest.mark.parametrize("want_deadline", [False, True])
def test_route_bin_wide_prompts(eng, restate, want_deadline):
    """K1b's fold reads 16-bit prompts straight from the sorted list when every prompt of a
    staging chunk fits 16 bits, else through stage indices: windows mixing both kinds (prompts
    up to INT32_MAX, zero and negative) must give the same bits as the oracle."""
    api = _api()
    profs = synth_profiles(api)[:4]
    eng.set_profiles(profs)
    a, p, _ = restate.gen_poisson_trace(5.0, 1_800_000, 768.0, 3072.0, 0.15, 128.0, seed=5)
    rng = np.random.default_rng(5)
    wms = 60_000
    w = a // wms
    wide = (w % 3) == 1  # every third window: some prompts beyond 16 bits
    pick = wide & (rng.random(len(p)) < 0.2)
    p = p.copy()
    p[pick] = rng.integers(65_536, 2**31 - 1, int(pick.sum()))
    p[wide & (rng.random(len(p)) < 0.05)] = 65_535
    neg = (w % 3 == 2) & (rng.random(len(p)) < 0.02)
    p[neg] = rng.integers(-(2**31), 1, int(neg.sum()))
    thr = [128, 256, 512, 768, 1024, 2048, 4096]
    nw = int(a[-1] // wms) + 1
    rr = eng.route_bin(a, p, api.RoutingConfig(True, thr, list(range(len(thr) + 1))), wms, 0, nw,
                       want_deadline=want_deadline)
    torch.cuda.synchronize()
    cls, cnt, tref, mdl, _ = restate.route_bin(a, p, thr, wms, 0, nw, [to_oracle(x) for x in profs])
    np.testing.assert_array_equal(rr.cls.cpu().numpy(), cls)
    np.testing.assert_array_equal(rr.count.cpu().numpy().view(np.uint32), cnt)
    np.testing.assert_array_equal(u64(rr.t_ref.cpu().numpy()), u64(tref))
    if want_deadline:
        np.testing.assert_array_equal(u64(rr.min_deadline.cpu().numpy()), u64(mdl))
    eng.set_profiles([api.GpuProfile.default_profile()])


def test_route_bin_edges(eng, restate):
    """empty windows, a window offset (w0), requests outside the range, routing disabled."""
    api = _api()
    eng.set_profiles([api.GpuProfile.default_profile()])
    a = np.array([0, 5, 5, 70_000, 70_001, 250_000, 250_000, 250_001], np.int64)
    p = np.array([10, 1024, 1025, 4096, 1, 600, 2000, 3], np.int32)
    prof = to_oracle(api.GpuProfile.default_profile())
    for thr, enabled in (([1024], True), ([1024], False)):
        rr = eng.route_bin(a, p, api.RoutingConfig(enabled, thr, [0, 1]), 60_000, 1, 4,
                           want_deadline=True, want_fifo=True)
        torch.cuda.synchronize()
        got_cnt = rr.count.cpu().numpy().view(np.uint32)
        o = restate.route_bin(a, p, thr if enabled else [], 60_000, 1, 4, [prof])
        np.testing.assert_array_equal(got_cnt, o[1])
        np.testing.assert_array_equal(u64(rr.t_ref.cpu().numpy()), u64(o[2]))
        inside = slice(3, 8)
        np.testing.assert_array_equal(rr.cls.cpu().numpy()[inside], o[0][inside])


@pytest.mark.parametrize("mode", ["fixed", "slack"])
def test_prefill_select_matches_oracle(eng, restate, mode):
    api = _api()
    profs = synth_profiles(api)
    eng.set_profiles(profs)
    thr = [256, 512, 1024, 2048]
    a, p, _ = restate.gen_poisson_trace(6.0, 3_600_000, 1024.0, 6144.0, 0.35, 32.0, seed=5)
    wms = 60_000
    nw = int(a[-1] // wms) + 1
    rr = eng.route_bin(a, p, api.RoutingConfig(True, thr, list(range(5))), wms, 0, nw,
                       want_deadline=True)
    qcfg = api.QueueOptimizerConfig()
    if mode == "fixed":
        sel = eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=0.95 * wms)
    else:
        sel = eng.prefill_select(rr, api.L.DEADLINE_SLACK, qopt=qcfg)
    torch.cuda.synchronize()
    cls, cnt, tref, mdl, _ = restate.route_bin(a, p, thr, wms, 0, nw, [to_oracle(x) for x in profs],
                                               fifo=False)
    fi = sel.f_idx.cpu().numpy()
    en = sel.energy_j.cpu().numpy()
    win = sel.window_ms.cpu().numpy()
    n_inf = 0
    for pi, pr in enumerate(profs):
        op = to_oracle(pr)
        for c in range(len(cnt)):
            if cnt[c] == 0:
                assert fi[pi, c] == -2
                continue
            if mode == "fixed":
                W = 0.95 * wms
            else:
                now = float((c // 5) * wms)
                slack = mdl[c] - now
                W = max(qcfg.margin_prefill * slack, qcfg.min_budget_ms) \
                    if not (qcfg.margin_prefill * slack < qcfg.min_budget_ms) else qcfg.min_budget_ms
                W = qcfg.min_budget_ms if qcfg.margin_prefill * slack < qcfg.min_budget_ms \
                    else qcfg.margin_prefill * slack
                assert u64(win[c]) == u64(W)
            r = restate.select_t(op, tref[pi, c], W)
            if r is None:
                n_inf += 1
                assert fi[pi, c] == -1
            else:
                assert fi[pi, c] == r[0] and u64(en[pi, c]) == u64(r[2]), (pi, c)
    assert n_inf > 0  # the long classes are over-subscribed: infeasible cells exercised
    eng.set_profiles([api.GpuProfile.default_profile()])


def test_rounding_driven_argmin_probes_on_gpu(eng):
    api = _api()
    prof = api.GpuProfile.default_profile()
    b = api.PrefillBatch([api.PrefillJob(0, 1024)])
    for D, f, e in [(1e12, 975.0, 15000000066.645506), (1e15, 975.0, 15000000000066.645),
                    (1e17, 945.0, 1500000000000066.8), (1e20, 390.0, 1.5e18),
                    (1e300, 210.0, 1.5e298)]:
        ch = eng.select_frequency(b, D, prof)
        assert ch.f_mhz == f and ch.energy_j == e
    batch = api.PrefillBatch([api.PrefillJob(i, L) for i, L in enumerate([512, 700, 300, 2048])])
    assert eng.select_frequency(batch, 100.0, prof) is None
    ch = eng.select_frequency(batch, 1000.0, prof)
    assert (ch.f_mhz, ch.energy_j) == (975.0, 260.74498153855995)
    ch = eng.select_frequency(batch, 57000.0, prof)
    assert (ch.f_mhz, ch.energy_j) == (975.0, 1100.74498153856)
    # frozen 313.803221 J case (proj/tests/test_prefill_opt.cpp:67-83)
    p2 = api.GpuProfile("t", prof.grid, api.LatencyModel(0.0, 1.0, 0.0, 1410.0), prof.decode,
                        api.PowerModel(1e-9, 0.0, 0.1, 50.0, 60.0))
    e = eng.energy_total(api.PrefillBatch([api.PrefillJob(0, 1000)]), 1410.0, 3000.0, p2)
    assert e.feasible and abs(e.total_j - 313.803221) / 313.803221 < 1e-9
    with pytest.raises(api.ModelError):
        eng.energy_total(api.PrefillBatch([]), 1410.0, 3000.0, prof)
    with pytest.raises(api.ModelError):
        eng.energy_total(batch, 1411.0, 3000.0, prof)
    eng.set_profiles([prof])


def test_acceptance_batches_vs_reference(eng, ref, prof):
    """acceptance check 2 shape (acceptance_main.cpp:149-188) + running jobs + random power
    shapes: GPU select/energy == the reference library, bit for bit."""
    api = _api()
    rng = np.random.default_rng(2)
    gp = api.GpuProfile.default_profile()
    for shape in range(4):
        if shape:
            gp = api.GpuProfile("r", gp.grid, api.LatencyModel(1e-6 + 1e-4 * rng.random(),
                                                              0.5 * rng.random(), 20 * rng.random(),
                                                              1410.0), gp.decode,
                                api.PowerModel(1e-8 + 4e-7 * rng.random(), -2e-4 * rng.random(),
                                               0.2 * rng.random(), 50 + 400 * rng.random(),
                                               80.0 * rng.random() + 1e-3))
            try:
                gp.validate()
            except api.ModelError:
                continue
        op = to_oracle(gp)
        nb = 1000
        sizes = rng.integers(1, 7, nb)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        prompts = rng.integers(16, 6000, off[-1]).astype(np.int32)
        wf = np.where(rng.random(off[-1]) < 0.2, rng.random(off[-1]), 1.0)
        win = np.where(np.arange(nb) % 10 == 9, 0.5 + 30 * rng.random(nb), 10 + 4000 * rng.random(nb))
        f_idx, en, _, tr = eng.select_batches(off, prompts, win, gp, wf)
        grid = np.array(gp.grid.frequencies())
        fsel = grid[rng.integers(0, len(grid), nb)]
        busy, act, idl, tot, feas = eng.energy_batches(off, prompts, fsel, win, gp, wf)
        torch.cuda.synchronize()
        fi, en, tr = f_idx.cpu().numpy(), en.cpu().numpy(), tr.cpu().numpy()
        act, idl, tot, feas = act.cpu().numpy(), idl.cpu().numpy(), tot.cpu().numpy(), feas.cpu().numpy()
        rf, re_, found = ref.select_many(op, off, prompts, win, wf)
        n_inf = 0
        for b in range(nb):
            s, e = off[b], off[b + 1]
            assert u64(tr[b]) == u64(ref.t_ref(op, prompts[s:e], wf[s:e]))
            if not found[b]:
                n_inf += 1
                assert fi[b] == -1
            else:
                assert grid[fi[b]] == rf[b] and u64(en[b]) == u64(re_[b]), b
            ra = ref.energy_total(op, prompts[s:e], fsel[b], win[b], wf[s:e])
            assert (act[b], idl[b], tot[b], bool(feas[b])) == ra, b
        assert n_inf > 0


def test_online_snapshots_reproduce_reference_commands(eng, ref, prof):
    """C1: the reference simulator's own optimizer snapshots (greenllm, Alibaba-shaped 1 h,
    3 classes; captured at simkernel.cpp:487) replayed on the GPU give the reference's
    PrefillFreqCommands exactly (clock, window, infeasible flag)."""
    api = _api()
    a, p, o = ref.gen_poisson_trace(5.0, 3_600_000, seed=7)
    r = ref.run_capture(a, p, o, prof, "greenllm", thresholds=(512, 1024), worker_map=(0, 1, 2))
    off = r["snap_off"]
    nonempty = np.diff(off) > 0
    idx = np.nonzero(nonempty)[0]
    # CSR over the non-empty snapshots
    sizes = np.diff(off)[idx]
    noff = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    sel = np.concatenate([np.arange(off[i], off[i + 1]) for i in idx])
    gp = api.GpuProfile.default_profile()
    f_idx, en, win, _ = eng.select_batches(noff, r["job_prompt"][sel], None, gp, r["job_wf"][sel],
                                           api.L.DEADLINE_SLACK, 0.0, r["job_deadline"][sel],
                                           r["snap_now"][idx], api.QueueOptimizerConfig())
    torch.cuda.synchronize()
    fi = f_idx.cpu().numpy()
    win = win.cpu().numpy()
    f = np.where(fi >= 0, 210.0 + 15.0 * fi, 1410.0)
    assert len(idx) == len(r["cmd_f"]) and len(idx) > 30_000
    np.testing.assert_array_equal(r["snap_class"][idx], r["cmd_class"])
    np.testing.assert_array_equal(f, r["cmd_f"])
    np.testing.assert_array_equal(u64(win), u64(r["cmd_window"]))
    np.testing.assert_array_equal((fi < 0).astype(np.uint8), r["cmd_infeasible"])
    assert r["cmd_infeasible"].sum() > 1000


def test_online_snapshots_work_fraction_on_device(eng, ref, restate, prof):
    """a5: the running prefill job's work_fraction computed ON THE DEVICE from the raw worker
    state (remaining_ref, updated_ms, applied clock, t_ref; simkernel.cpp:476-479), as the
    (reference-pinned) restated simulator records it at every optimizer tick of the C1 run:
    the device's T_ref bits equal the host-side fraction's, and the commands equal the ones
    the unmodified reference simulator issued."""
    api = _api()
    from oracle import oracle as O
    a, p, o = ref.gen_poisson_trace(5.0, 3_600_000, seed=7)
    r = ref.run_capture(a, p, o, prof, "greenllm", thresholds=(512, 1024), worker_map=(0, 1, 2))
    pol = O.PolicyHolder("greenllm", thresholds=(512, 1024), worker_map=(0, 1, 2))
    sn = restate.sim_run(prof, pol, O.default_slo(), O.default_sim_cfg(n_prefill_workers=3),
                         a, p, o)["snapshots"]
    assert len(sn["now"]) == len(r["cmd_f"]) and sn["running"].sum() > 10_000
    gp = api.GpuProfile.default_profile()
    running = {"running": sn["running"], "remaining_ref_ms": sn["rem_ref"],
               "updated_ms": sn["upd_ms"], "freq_mhz": sn["freq"], "t_ref_ms": sn["t_ref"]}
    f_idx, en, win, t_dev = eng.select_batches(sn["off"], sn["prompt"], None, gp, None,
                                               api.L.DEADLINE_SLACK, 0.0, sn["deadline"],
                                               sn["now"], api.QueueOptimizerConfig(),
                                               running=running)
    # the same batches with the host-computed fractions: identical T_ref bits
    _, _, _, t_host = eng.select_batches(sn["off"], sn["prompt"], None, gp, sn["wf"],
                                         api.L.DEADLINE_SLACK, 0.0, sn["deadline"], sn["now"],
                                         api.QueueOptimizerConfig())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u64(t_dev.cpu().numpy()), u64(t_host.cpu().numpy()))
    fi = f_idx.cpu().numpy()
    f = np.where(fi >= 0, 210.0 + 15.0 * fi, 1410.0)
    np.testing.assert_array_equal(sn["cls"], r["cmd_class"])
    np.testing.assert_array_equal(f, r["cmd_f"])
    np.testing.assert_array_equal(u64(win.cpu().numpy()), u64(r["cmd_window"]))
    np.testing.assert_array_equal((fi < 0).astype(np.uint8), r["cmd_infeasible"])


def test_band_tables_vs_reference(eng, ref):
    api = _api()
    rng = np.random.default_rng(3)
    base = api.GpuProfile.default_profile()
    profs, t_slo, workers = [], [], []
    for i in range(64):
        d = base.decode
        p = api.GpuProfile("b", base.grid, base.prefill,
                           api.DecodeStepModel(d.alpha0_ms * (0.5 + rng.random()), d.alpha1_ms,
                                               d.beta0_ms, d.beta1_ms * (0.5 + rng.random()),
                                               1410.0), base.power)
        profs.append(p)
        t_slo.append(40 + 120 * rng.random())
        workers.append(int(rng.integers(1, 9)))
    lo, hi, fo, fe = eng.build_band_tables(profs, np.arange(64), t_slo, workers, [64] * 64, LEVELS)
    lo, hi, fo, fe = (x.cpu().numpy() for x in (lo, hi, fo, fe))
    for i in range(64):
        want = ref.band_table(to_oracle(profs[i]), LEVELS, t_slo[i], workers[i], 64)
        np.testing.assert_array_equal(u64(lo[i]), u64(want[0]))
        np.testing.assert_array_equal(u64(hi[i]), u64(want[1]))
        np.testing.assert_array_equal(fo[i], want[2])
        np.testing.assert_array_equal(fe[i].astype(bool), want[3])
    t = eng.build_band_table(base, LEVELS, 95.0, 4, 64)
    assert [b.f_opt_mhz for b in t.buckets] == [210, 210, 210, 210, 225, 240, 255, 270, 285, 300,
                                                315, 315, 330, 360, 390]
    with pytest.raises(api.ModelError):
        eng.build_band_table(base, [200.0, 200.0], 95.0, 4, 64)


def _telemetry(rng, S, t_end, rate_hz=200.0):
    offs, ts, toks, goffs, gaps = [0], [], [], [0], []
    for s in range(S):
        n = int(t_end / 1000.0 * rate_hz * (0.5 + rng.random()))
        t = np.sort(rng.uniform(0.0, t_end, n))
        k = rng.integers(0, n, n // 10)
        t[k] = np.round(t[k] / 20.0) * 20.0  # events exactly on tick times
        t = np.sort(t)
        ts.append(t)
        toks.append(rng.integers(1, 12, n).astype(np.int32))
        ng = rng.integers(0, 12, n)
        for g in ng:
            goffs.append(goffs[-1] + int(g))
        gaps.append(rng.gamma(4.0, 20.0, int(ng.sum())))
        offs.append(offs[-1] + n)
    api = _api()
    return api.Telemetry(np.array(offs, np.int64), np.concatenate(ts), np.concatenate(toks),
                         np.array(goffs, np.int64), np.concatenate(gaps))


def _stream_arrays(tel, s):
    e0, e1 = tel.ev_off[s], tel.ev_off[s + 1]
    goff = tel.gap_off[e0:e1 + 1]
    return TelemetryArrays(tel.t_ms[e0:e1].copy(), tel.tokens[e0:e1].copy(),
                           (goff - goff[0]).astype(np.int64), tel.gaps[goff[0]:goff[-1]].copy())


@pytest.mark.parametrize("cap", [1, 16, 256])
def test_window_series_matches_oracle(eng, restate, cap):
    rng = np.random.default_rng(cap)
    tel = _telemetry(rng, 6, 12_000.0)
    has, p95, tps = eng.window_series(tel, cap, 20.0, 200.0, 12_000.0)
    torch.cuda.synchronize()
    for s in range(tel.n_streams):
        h, p, t = restate.window_series(_stream_arrays(tel, s), cap, 20.0, 200.0, 12_000.0)
        np.testing.assert_array_equal(has[s].cpu().numpy(), h)
        np.testing.assert_array_equal(u64(p95[s].cpu().numpy()), u64(p))
        np.testing.assert_array_equal(u64(tps[s].cpu().numpy()), u64(t))


def test_decode_replay_matches_oracle_full_records(eng, restate):
    """Param sweep (hysteresis x step x TBT target) on shared telemetry: every DecisionRecord
    bit-identical to the restated DecodeController driven exactly like Sim."""
    api = _api()
    rng = np.random.default_rng(9)
    t_end = 30_000.0
    tel = _telemetry(rng, 4, t_end)
    gp = api.GpuProfile.default_profile()
    cfgs, table_of, stream_of, worker = [], [], [], []
    tslos = [60.0, 95.0, 130.0]
    for h in (1, 3, 5):
        for st in (15.0, 30.0):
            for ti, ts in enumerate(tslos):
                for s in range(4):
                    cfgs.append(api.DecodeCtlConfig(tslo_ms=ts, step_mhz=st,
                                                    max_step_mhz=max(30.0, st),
                                                    hysteresis_count=h))
                    table_of.append(ti)
                    stream_of.append(s)
                    worker.append(s)
    lo, hi, fo, fe = eng.build_band_tables([gp], [0] * 3, [t * 0.95 for t in tslos], [4] * 3,
                                           [64] * 3, LEVELS)
    has, p95, tps = eng.window_series(tel, 256, 20.0, 200.0, t_end)
    cap = 2048
    out = eng.decode_replay(cfgs, table_of, stream_of, worker, lo, hi, fo, gp.grid, has, p95, tps,
                            t_end, rec_cap=cap)
    torch.cuda.synchronize()
    lo_h, hi_h, fo_h = (x.cpu().numpy() for x in (lo, hi, fo))
    nrec = out["n_rec"].cpu().numpy()
    dig = out["digest"].cpu().numpy().view(np.uint64)
    recs = out["records"].cpu().numpy()
    for n, c in enumerate(cfgs):
        oc = default_ctl_cfg(tslo_ms=c.tslo_ms, step_mhz=c.step_mhz, max_step_mhz=c.max_step_mhz,
                             hysteresis_count=c.hysteresis_count)
        tb = band_table(lo_h[table_of[n]], hi_h[table_of[n]], fo_h[table_of[n]])
        want = restate.replay_telemetry(oc, tb, 210.0, 1410.0, worker[n],
                                        _stream_arrays(tel, stream_of[n]), t_end)
        assert nrec[n] == len(want)
        assert dig[n] == restate.digest(want)
        got = recs[n, :min(cap, len(want))].reshape(-1).view(want.dtype)
        assert (got == want[:cap]).all(), n


def test_fine_loop_threshold_edges(eng, restate):
    """p95 values within a few ulps of upper*den and lower*den: the division-free margin test
    of K3b must take exactly the reference's decisions (decode_ctl.cpp:150-157)."""
    api = _api()
    gp = api.GpuProfile.default_profile()
    rng = np.random.default_rng(13)
    cfgs, series = [], []
    for it in range(48):
        tslo = float(rng.uniform(40.0, 160.0))
        margin = float(rng.choice([0.6, 0.95, 1.0, 1.3, float(rng.uniform(0.2, 2.0))]))
        c = api.DecodeCtlConfig(tslo_ms=tslo, margin_decode=margin, coarse_period_ms=1e9,
                                adapt_period_s=1e9, tps_scale=1.0)
        den = margin * tslo
        vals = []
        for thr in (c.upper_margin, c.lower_margin):
            base = thr * den
            for k in range(-4, 5):
                vals.append(np.nextafter(base, np.inf * k) if k else base)
                v = base
                for _ in range(abs(k)):
                    v = np.nextafter(v, np.inf if k > 0 else -np.inf)
                vals.append(v)
        vals = np.array(vals)
        rng.shuffle(vals)
        cfgs.append(c)
        series.append(vals)
    nf = max(len(v) for v in series)
    t_end = 20.0 * nf
    has = np.ones((len(cfgs), nf), np.uint8)
    p95 = np.stack([np.resize(v, nf) for v in series])
    tps = np.zeros((len(cfgs), 1))
    one = band_table([0.0], [math.inf], [705.0])
    lo, hi, fo = np.array([[0.0]]), np.array([[math.inf]]), np.array([[705.0]])
    dev = lambda x, dt: torch.as_tensor(x, device="cuda").to(dt)
    out = eng.decode_replay(cfgs, [0] * len(cfgs), np.arange(len(cfgs)), [0] * len(cfgs), lo, hi,
                            fo, gp.grid, dev(has, torch.uint8), dev(p95, torch.float64),
                            dev(tps, torch.float64), t_end, rec_cap=nf + 4)
    torch.cuda.synchronize()
    recs = out["records"].cpu().numpy()
    for n, c in enumerate(cfgs):
        oc = default_ctl_cfg(tslo_ms=c.tslo_ms, margin_decode=c.margin_decode,
                             coarse_period_ms=1e9, adapt_period_s=1e9, tps_scale=1.0)
        want = restate.replay_series(oc, one, 210.0, 1410.0, 0, has[n], p95[n], tps[n], t_end)
        got = recs[n, :len(want)].reshape(-1).view(want.dtype)
        assert int(out["n_rec"][n].item()) == len(want)
        assert (got == want).all(), n


def test_decode_replay_reproduces_reference_closed_loop_run(eng, ref, prof):
    """The reference simulator's own controllers (greenllm, sinusoid decode load): their
    captured per-tick inputs replayed on the GPU give the reference's decision log."""
    api = _api()
    a, p, o = ref.gen_sinusoid_decode_trace(1500.0, 1000.0, 120000.0, 150000, 11)
    r = ref.run_capture(a, p, o, prof, "greenllm")
    gp = api.GpuProfile.default_profile()
    cfg = api.DecodeCtlConfig()
    lo, hi, fo, fe = eng.build_band_tables([gp], [0], [cfg.tslo_ms * cfg.margin_decode], [4], [64],
                                           LEVELS)
    t_end = float(r["fine_t"][-1])
    nf = eng.lib.gsb_n_ticks(20.0, t_end)
    nc = eng.lib.gsb_n_ticks(200.0, t_end)
    has = np.zeros((4, nf), np.uint8)
    p95 = np.zeros((4, nf))
    tps = np.zeros((4, nc))
    for w in range(4):
        m, mc = r["fine_worker"] == w, r["coarse_worker"] == w
        has[w], p95[w], tps[w] = r["fine_has"][m], r["fine_p95"][m], r["coarse_tps"][mc]
    dev = lambda x, dt: torch.as_tensor(x, device="cuda").to(dt)
    out = eng.decode_replay([cfg] * 4, [0] * 4, range(4), range(4), lo, hi, fo, gp.grid,
                            dev(has, torch.uint8), dev(p95, torch.float64),
                            dev(tps, torch.float64), t_end, rec_cap=12_000)
    torch.cuda.synchronize()
    dec = r["decisions"]
    recs = out["records"].cpu().numpy()
    for w in range(4):
        want = dec[dec["worker"] == w]
        n = int(out["n_rec"][w].item())
        assert n == len(want)
        got = recs[w, :n].reshape(-1).view(want.dtype)
        assert (got == want).all()


@pytest.mark.parametrize("thr", [[512, 1024], [256, 512, 1024, 2048],
                                 [128, 256, 512, 768, 1024, 2048, 4096]])
def test_fused_select_summary_equals_standalone(eng, restate, thr):
    """gsb_prefill_select_summary (K2 + the per-class reduction in one launch) gives the same
    per-cell decisions as gsb_prefill_select and the same summary BYTES as
    gsb_prefill_summary; counts / min are exact against a host recount."""
    api = _api()
    profs = synth_profiles(api)
    eng.set_profiles(profs)
    C = len(thr) + 1
    a, p, _ = restate.gen_poisson_trace(5.0, 5_400_000, seed=21)
    rr = eng.route_bin(a, p, api.RoutingConfig(True, thr, list(range(C))), 45_000)
    ref = eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=0.95 * 45_000)
    summ = eng.summary_buffer(C)
    for _ in range(3):  # repeated launches agree
        sel = eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=0.95 * 45_000,
                                 summary_out=summ)
        fused = summ.cpu().numpy().view(eng.SUMMARY_DTYPE).reshape(len(profs), C)
        assert torch.equal(sel.f_idx, ref.f_idx)
        assert torch.equal(sel.energy_j.view(torch.int64), ref.energy_j.view(torch.int64))
        std = eng.prefill_summary(sel, C)
        assert fused.tobytes() == std.tobytes()
    fi = sel.f_idx.cpu().numpy()
    en = sel.energy_j.cpu().numpy()
    for pi in range(len(profs)):
        f2, e2 = fi[pi].reshape(-1, C), en[pi].reshape(-1, C)
        for c in range(C):
            s = fused[pi, c]
            assert s["n_empty"] == (f2[:, c] == -2).sum()
            assert s["n_cmd"] == (f2[:, c] != -2).sum()
            assert s["n_infeasible"] == (f2[:, c] == -1).sum()
            ok = f2[:, c] >= 0
            if ok.any():
                e = e2[ok, c]
                assert abs(s["sum_energy_j"] - e.sum()) <= 1e-11 * abs(e.sum())
                k = int(np.argmin(np.where(ok, e2[:, c], np.inf)))
                assert s["min_energy_j"] == e2[k, c] and s["argmin_cell"] == k * C + c
            else:
                assert s["argmin_cell"] == -1


@pytest.mark.parametrize("mode,n_prof,minutes,thr", [
    ("deadline", 1, 7, [1024]),          # DEADLINE_SLACK, one profile, 7 windows (< one tile)
    ("fixed", 2, 301, []),               # routing disabled (C = 1), tile tail of 45 cells
    ("fixed", 3, 90, [256, 512, 1024, 2048]),
])
def test_fused_summary_modes_and_shapes(eng, restate, mode, n_prof, minutes, thr):
    """The fused K2 + summary path on small / ragged shapes, DEADLINE_SLACK windows, 1-3
    profiles and routing off: per-cell results equal the unfused kernel, summary bytes equal
    gsb_prefill_summary."""
    api = _api()
    profs = synth_profiles(api)[:n_prof]
    eng.set_profiles(profs)
    C = len(thr) + 1
    a, p, _ = restate.gen_poisson_trace(2.0, minutes * 60_000, seed=5 + minutes)
    routing = api.RoutingConfig(bool(thr), thr or [1024], list(range(C)) if thr else [0, 0])
    rr = eng.route_bin(a, p, routing, 60_000, want_deadline=(mode == "deadline"))
    kw = dict(fixed_window_ms=0.95 * 60_000) if mode == "fixed" else {}
    m = api.L.FIXED_WINDOW if mode == "fixed" else api.L.DEADLINE_SLACK
    ref = eng.prefill_select(rr, m, **kw)
    summ = eng.summary_buffer(rr.n_classes)
    sel = eng.prefill_select(rr, m, summary_out=summ, **kw)
    assert torch.equal(sel.f_idx, ref.f_idx)
    assert torch.equal(sel.energy_j.view(torch.int64), ref.energy_j.view(torch.int64))
    busy = rr.count.view(torch.int32) != 0  # PrefillFreqCommand::window_ms exists per command
    assert torch.equal(sel.window_ms.view(torch.int64)[busy], ref.window_ms.view(torch.int64)[busy])
    fused = summ.cpu().numpy().view(eng.SUMMARY_DTYPE).reshape(n_prof, rr.n_classes)
    assert fused.tobytes() == eng.prefill_summary(sel, rr.n_classes).tobytes()
    assert int(fused["n_cmd"].sum() + fused["n_empty"].sum()) == n_prof * rr.n_cells


def test_summary_is_deterministic_and_exact_counts(eng, restate):
    api = _api()
    eng.set_profiles([api.GpuProfile.default_profile()])
    a, p, _ = restate.gen_poisson_trace(5.0, 7_200_000, seed=3)
    rr = eng.route_bin(a, p, api.RoutingConfig(True, [512, 1024], [0, 1, 2]), 60_000)
    sel = eng.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=0.95 * 60_000)
    s1 = eng.prefill_summary(sel, 3)
    s2 = eng.prefill_summary(sel, 3)
    assert s1.tobytes() == s2.tobytes()
    fi = sel.f_idx.cpu().numpy()[0].reshape(-1, 3)
    en = sel.energy_j.cpu().numpy()[0].reshape(-1, 3)
    for c in range(3):
        assert s1[0, c]["n_empty"] == (fi[:, c] == -2).sum()
        assert s1[0, c]["n_infeasible"] == (fi[:, c] == -1).sum()
        e = en[fi[:, c] >= 0, c]
        assert abs(s1[0, c]["sum_energy_j"] - e.sum()) <= 1e-9 * abs(e.sum())
        assert s1[0, c]["min_energy_j"] == e.min()


@pytest.mark.parametrize("want_deadline", [False, True])
def test_route_bin_reads_pinned_host_arrivals_in_place(eng, restate, want_deadline):
    """A pinned host arrival tensor is read in place by K1 (zero copy over PCIe): every output
    equals the device-resident path's, bit for bit."""
    api = _api()
    profs = synth_profiles(api)[:4]
    eng.set_profiles(profs)
    a, p, _ = restate.gen_poisson_trace(6.0, 3_600_000, 768.0, 3072.0, 0.15, 128.0, seed=8)
    thr = [128, 256, 512, 768, 1024, 2048, 4096]
    rc = api.RoutingConfig(True, thr, list(range(len(thr) + 1)))
    nw = int(a[-1] // 60_000) + 1
    h = torch.as_tensor(a).pin_memory()
    assert h.is_pinned()
    r_dev = eng.route_bin(torch.as_tensor(a, device="cuda"), p, rc, 60_000, 0, nw,
                          want_deadline=want_deadline)
    r_host = eng.route_bin(h, p, rc, 60_000, 0, nw, want_deadline=want_deadline)
    torch.cuda.synchronize()
    for f in ("bounds", "cls", "count", "t_ref", "n_nonempty"):
        assert torch.equal(getattr(r_dev, f), getattr(r_host, f)), f
    n = int(r_dev.n_nonempty.item())  # list entries past n are not written
    assert torch.equal(r_dev.nonempty[:n], r_host.nonempty[:n])
    assert torch.equal(r_dev.t_ref_list[:, :n], r_host.t_ref_list[:, :n])
    if want_deadline:
        assert torch.equal(r_dev.min_deadline.view(torch.int64), r_host.min_deadline.view(torch.int64))
    eng.set_profiles([api.GpuProfile.default_profile()])
