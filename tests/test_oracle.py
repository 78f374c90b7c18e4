"""Pins the CPU oracle (oracle/gs_oracle.c) before anything is checked against it:
(1) the reference's golden values (the reference's own tests), and
(2) element-wise equality with the unmodified reference library (oracle/_ref)."""
import math

import numpy as np
import pytest

from oracle.oracle import (ACTIONS, CtlCfg, Profile, TelemetryArrays, band_table, default_ctl_cfg,
                           default_qopt_cfg)

LEVELS = np.arange(200.0, 3000.0 + 1e-9, 200.0)


def bits(x):
    return np.float64(x).view(np.uint64)


# ----------------------------------------------------------------- golden values
def test_model_golden_values(restate, prof):
    # proj/tests/test_simkernel.cpp:83-101, proj/tests/python/test_smoke.py:24-32
    assert restate.validate(prof)
    assert restate.t_ref(prof, [512]) == pytest.approx(74.68288, rel=1e-12)
    assert restate.active_power(prof, 1410.0) == pytest.approx(536.70536, rel=1e-12)
    assert restate.active_power(prof, 900.0) == pytest.approx(297.14, rel=1e-12)
    g = restate.grid(prof)
    assert len(g) == 81 and g[0] == 210.0 and g[-1] == 1410.0
    ok, b, tbt = restate.steady_state(prof, 1.0, 1410.0, 64)
    assert ok and b == 1.0 and tbt == pytest.approx(23.735, rel=1e-12)


def test_frozen_window_energy(restate):
    # proj/tests/test_prefill_opt.cpp:67-83
    p = Profile(210.0, 1410.0, 15.0, 1410.0, 0.0, 1.0, 0.0, 1410.0, 14.5, 0.1, 9.0, 0.135, 1410.0,
                1e-9, 0.0, 0.1, 50.0, 60.0)
    a, i, t, feas = restate.energy_total(p, [1000], 1410.0, 3000.0)
    assert feas
    assert abs(t - 313.803221) / 313.803221 < 1e-9
    assert a == pytest.approx(193.803221, rel=1e-9) and i == pytest.approx(120.0, rel=1e-9)
    assert abs(restate.closed_form(p, [1000], 1410.0, 3000.0) - t) / t < 1e-9


@pytest.mark.parametrize("D,f,e", [
    (1e12, 975.0, 15000000066.645506), (1e15, 975.0, 15000000000066.645),
    (1e17, 945.0, 1500000000000066.8), (1e20, 390.0, 1.5e18), (1e300, 210.0, 1.5e298)])
def test_rounding_driven_argmin_probes(restate, prof, D, f, e):
    # fp64 rounding of the idle term moves the reference's argmin.
    idx, fo, eo = restate.select_frequency(prof, [1024], D)
    assert fo == f and eo == e


def test_select_frequency_golden(restate, prof):
    b = [512, 700, 300, 2048]
    assert restate.select_frequency(prof, b, 100.0) is None
    assert restate.select_frequency(prof, b, 400.0) is None
    assert restate.select_frequency(prof, b, 1000.0)[1:] == (975.0, 260.74498153855995)
    assert restate.select_frequency(prof, b, 57000.0)[1:] == (975.0, 1100.74498153856)
    # boundary: D == busy(705) is feasible at 705 (proj/tests/test_prefill_opt.cpp:85-94)
    busy = restate.t_ref(prof, [1024]) * 1410.0 / 705.0
    a, i, t, feas = restate.energy_total(prof, [1024], 705.0, busy)
    assert feas and i == 0.0
    assert not restate.energy_total(prof, [1024], 705.0, busy * 0.5)[3]


def test_queue_tick_semantics(restate, prof):
    # proj/tests/test_prefill_opt.cpp:188-234
    cfg = default_qopt_cfg()
    f, w, inf, idx, e = restate.queue_tick_one(prof, cfg, [1024], [1e12], 0.0)
    assert not inf and f == restate.select_frequency(prof, [1024], 1e15)[1]
    f, w, inf, idx, e = restate.queue_tick_one(prof, cfg, [4096], [-500.0], 0.0)
    assert w == cfg.min_budget_ms and f == 1410.0 and inf
    small = default_qopt_cfg(margin_prefill=0.2, min_budget_ms=1.0)
    f1, w1, *_ = restate.queue_tick_one(prof, small, [2048], [400.0], 0.0)
    assert w1 == pytest.approx(80.0)
    f2, *_ = restate.queue_tick_one(prof, default_qopt_cfg(margin_prefill=2.0), [2048], [400.0], 0.0)
    assert f2 <= f1


def test_classify_boundaries(restate):
    # proj/tests/test_router.cpp:19-32
    assert restate.classify([1024], 512) == 0
    assert restate.classify([1024], 1024) == 0
    assert restate.classify([1024], 1025) == 1
    assert restate.classify([256, 1024, 4096], 256) == 0
    assert restate.classify([256, 1024, 4096], 257) == 1
    assert restate.classify([256, 1024, 4096], 4097) == 3


def test_band_table_frozen(restate, prof):
    # proj/tests/test_decode_ctl.cpp:75-104
    lo, hi, fo, fe = restate.band_table(prof, LEVELS, 95.0, 4, 64)
    assert list(fo) == [210, 210, 210, 210, 225, 240, 255, 270, 285, 300, 315, 315, 330, 360, 390]
    assert fe.all() and lo[0] == 0.0 and hi[0] == 300.0 and math.isinf(hi[-1])


def test_quantile_nearest_rank(restate):
    # proj/tests/test_metrics.cpp:38-63
    v = np.arange(1, 101, dtype=np.float64)
    assert restate.quantile(v, 0.95) == 95.0 and restate.quantile(v, 0.99) == 99.0
    assert restate.quantile(v, 0.0) == 1.0 and restate.quantile(v, 1.0) == 100.0
    w = np.array([50.0] * 20 + [150.0])
    assert restate.quantile(w, 0.95) == 50.0


def _one_bucket(f):
    return band_table([0.0], [math.inf], [f])


def _two_buckets(split, flo, fhi):
    return band_table([0.0, split], [split, math.inf], [flo, fhi])


def test_fine_loop_sequence(restate):
    # proj/tests/test_decode_ctl.cpp:174-197: 705 -> 720 -> 720 -> 720 -> 705 -> 690 -> 690
    cfg = default_ctl_cfg(margin_decode=1.0, tps_scale=1.0, coarse_period_ms=1e9,
                          adapt_period_s=1e9)
    has = np.array([0, 1, 1, 1, 1, 1, 1], np.uint8)
    p95 = np.array([0, 120.0, 120.0, 80.0, 50.0, 50.0, 50.0])
    recs = restate.replay_series(cfg, _one_bucket(705.0), 210.0, 1410.0, 0, has, p95,
                                 np.zeros(0), 140.0)
    assert list(recs["command_mhz"]) == [705, 720, 720, 720, 705, 690, 690]
    assert [ACTIONS[a] for a in recs["action"]] == ["hold", "up", "up", "hold", "down", "down",
                                                    "down"]
    assert recs["p95_tbt_ms"][0] == 0.0 and recs["p95_tbt_ms"][1] == 120.0
    # CSV golden line 20,3,0,120,0,690,720,720,up (:365-373)
    r = restate.replay_series(cfg, _one_bucket(705.0), 210.0, 1410.0, 3, np.array([1], np.uint8),
                              np.array([120.0]), np.zeros(0), 20.0)[0]
    assert (r["tick_ms"], r["worker"], r["tps"], r["p95_tbt_ms"], r["bucket"], r["band_lo"],
            r["band_hi"], r["command_mhz"], ACTIONS[r["action"]]) == (
                20.0, 3, 0.0, 120.0, 0, 690.0, 720.0, 720.0, "up")


def test_coarse_hysteresis_sequence(restate):
    # proj/tests/test_decode_ctl.cpp:228-260 (coarse ticks only: fine/adapt pushed out)
    cfg = default_ctl_cfg(margin_decode=1.0, tps_scale=1.0, fine_period_ms=1e9,
                          adapt_period_s=1e9)
    tps = np.array([100.0, 100.0, 560.0, 100.0, 100.0, 100.0])
    recs = restate.replay_series(cfg, _two_buckets(500.0, 300.0, 600.0), 210.0, 1410.0, 0,
                                 np.zeros(0, np.uint8), np.zeros(0), tps, 1200.0)
    assert [ACTIONS[a] for a in recs["action"]] == [
        "coarse_pending", "coarse_pending", "coarse_hold", "coarse_pending", "coarse_pending",
        "coarse_commit"]
    assert recs["command_mhz"][-1] == 315.0


def test_windows_edges(ref, restate):
    # proj/tests/test_decode_ctl.cpp:154-172
    assert ref.tps_window(200.0, [0.0, 100.0, 250.0], [10, 20, 30], 300.0) == 50 * 1000.0 / 200.0
    assert ref.tbt_p95(4, [1, 2, 3, 4, 5, 6]) == 6.0
    tel = TelemetryArrays(np.array([0.0, 100.0, 250.0]), np.array([10, 20, 30], np.int32),
                          np.array([0, 0, 0, 0], np.int64), np.zeros(0))
    has, p95, tps = restate.window_series(tel, 4, 1e9, 150.0, 300.0)
    # coarse tick at 150 sees t=0,100 (0 >= 150-150); at 300 sees 250 and 100? 100 < 150 -> dropped
    assert list(tps) == [ref.tps_window(150.0, [0.0, 100.0], [10, 20], 150.0),
                         ref.tps_window(150.0, [0.0, 100.0, 250.0], [10, 20, 30], 300.0)]


# ----------------------------------------------------------------- vs the reference library
def test_generators_match_reference(ref, restate):
    for seed in (1, 7, 99):
        a = restate.gen_poisson_trace(5.0, 600_000, seed=seed)
        b = ref.gen_poisson_trace(5.0, 600_000, seed=seed)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
        a = restate.gen_poisson_trace(3.0, 600_000, 1024.0, 6144.0, 0.35, 32.0, seed)
        b = ref.gen_poisson_trace(3.0, 600_000, 1024.0, 6144.0, 0.35, 32.0, seed)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
    a = restate.gen_sinusoid_decode_trace(1500.0, 1000.0, 120000.0, 150000, 11)
    b = ref.gen_sinusoid_decode_trace(1500.0, 1000.0, 120000.0, 150000, 11)
    assert len(a[0]) == 1929
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_prefill_energy_and_argmin_vs_reference(ref, restate, prof):
    """Acceptance-style batches (acceptance_main.cpp:149-188) incl. tight windows, running
    jobs (work_fraction < 1) and random power shapes, bit-compared."""
    rng = np.random.default_rng(2)
    grid = restate.grid(prof)
    for it in range(1500):
        p = Profile(*prof.tuple())
        if it % 3 == 1:
            p.k3 = 1e-8 + 4e-7 * rng.random()
            p.k2 = -2e-4 * rng.random()
            p.k1 = 0.2 * rng.random()
            p.k0 = 50.0 + 400.0 * rng.random()
            p.p_idle_w = 80.0 * rng.random()
            p.lat_a, p.lat_b, p.lat_c = 1e-6 + 1e-4 * rng.random(), 0.5 * rng.random(), 20 * rng.random()
        n = int(rng.integers(1, 9))
        prompts = rng.integers(1, 8192, n).astype(np.int32)
        wf = rng.random(n) if it % 4 == 3 else None
        W = 0.5 + 30.0 * rng.random() if it % 10 == 9 else 10.0 + 4000.0 * rng.random()
        assert restate.t_ref(p, prompts, wf) == ref.t_ref(p, prompts, wf)
        f = float(grid[rng.integers(0, len(grid))])
        assert restate.energy_total(p, prompts, f, W, wf) == ref.energy_total(p, prompts, f, W, wf)
        assert bits(restate.closed_form(p, prompts, f, W, wf)) == bits(ref.closed_form(p, prompts, f, W, wf))
        got = restate.select_frequency(p, prompts, W, wf)
        want = ref.select_frequency(p, prompts, W, wf)
        assert (got is None) == (want is None)
        if got is not None:
            assert got[1:] == want


def test_queue_tick_vs_reference(ref, restate, prof):
    rng = np.random.default_rng(5)
    cfg = default_qopt_cfg()
    for it in range(300):
        nq = int(rng.integers(1, 5))
        sizes = rng.integers(0, 5, nq)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        prompts = rng.integers(16, 6000, off[-1]).astype(np.int32)
        now = float(rng.integers(0, 10_000_000))
        dl = now + rng.normal(300.0, 800.0, off[-1])
        wf = rng.random(off[-1])
        cmds = ref.queue_optimizer_tick(prof, cfg, np.arange(nq), off, prompts, dl, now, wf)
        mine = []
        for q in range(nq):
            s, e = off[q], off[q + 1]
            if s == e:
                continue
            f, w, inf, idx, en = restate.queue_tick_one(prof, cfg, prompts[s:e], dl[s:e], now, wf[s:e])
            mine.append((q, f, w, inf))
        assert mine == cmds


def test_dispatch_and_binning_vs_reference(ref, restate, prof):
    thr = [256, 512, 1024, 2048]
    a, p, o = ref.gen_poisson_trace(5.0, 1_800_000, 768.0, 3072.0, 0.15, 256.0, 3)
    q, fifo, sizes = ref.dispatch(thr, p)
    cls, cnt, tref, mdl, ff = restate.route_bin(a, p, thr, 3_600_000, 0, 1, [prof])
    np.testing.assert_array_equal(cls, q)           # queue assignment per request
    np.testing.assert_array_equal(ff, fifo)         # per-class FIFO order (one window)
    np.testing.assert_array_equal(cnt, sizes)
    # T_ref per cell equals the reference batch sum over the FIFO in order
    start = 0
    for c in range(len(thr) + 1):
        ids = fifo[start:start + sizes[c]]
        start += sizes[c]
        assert bits(tref[0, c]) == bits(ref.t_ref(prof, p[ids]))


def test_band_tables_vs_reference(ref, restate, prof):
    rng = np.random.default_rng(11)
    for it in range(60):
        p = Profile(*prof.tuple())
        p.dec_alpha0_ms *= 0.5 + rng.random()
        p.dec_beta1_ms *= 0.5 + rng.random()
        t_slo = 40.0 + 120.0 * rng.random()
        workers = int(rng.integers(1, 9))
        got = restate.band_table(p, LEVELS, t_slo, workers, 64)
        want = ref.band_table(p, LEVELS, t_slo, workers, 64)
        for x, y in zip(got, want):
            np.testing.assert_array_equal(x, y)


def _random_telemetry(rng, t_end, rate_hz=200.0):
    n = int(t_end / 1000.0 * rate_hz)
    t = np.sort(rng.uniform(0.0, t_end, n))
    t[rng.integers(0, n, n // 20)] = np.round(t[rng.integers(0, n, n // 20)] / 20.0) * 20.0
    t = np.sort(t)
    tok = rng.integers(1, 12, n).astype(np.int32)
    ng = rng.integers(0, 12, n)
    off = np.concatenate([[0], np.cumsum(ng)]).astype(np.int64)
    gaps = rng.gamma(4.0, 20.0, off[-1])
    return TelemetryArrays(t, tok, off, gaps)


def test_controller_replay_vs_reference(ref, restate, prof):
    rng = np.random.default_rng(17)
    for it in range(40):
        cfg = default_ctl_cfg(hysteresis_count=int(rng.integers(1, 6)),
                              step_mhz=float(rng.choice([15.0, 30.0])),
                              tslo_ms=float(rng.uniform(50, 150)),
                              tbt_window_tokens=int(rng.choice([16, 64, 256])))
        cfg.max_step_mhz = max(cfg.max_step_mhz, cfg.step_mhz)
        lo, hi, fo, fe = restate.band_table(prof, LEVELS, cfg.tslo_ms * cfg.margin_decode)
        tb = band_table(lo, hi, fo)
        tel = _random_telemetry(rng, 20_000.0)
        want = ref.replay_telemetry(cfg, tb, prof, it % 4, tel, 20_000.0)
        got = restate.replay_telemetry(cfg, tb, 210.0, 1410.0, it % 4, tel, 20_000.0)
        assert len(got) == len(want)
        assert (got == want).all()
        assert restate.digest(got) == ref.digest(want)
        has, p95, tps = restate.window_series(tel, cfg.tbt_window_tokens, cfg.fine_period_ms,
                                              cfg.coarse_period_ms, 20_000.0)
        ser = restate.replay_series(cfg, tb, 210.0, 1410.0, it % 4, has, p95, tps, 20_000.0)
        assert (ser == want).all()


def test_closed_loop_reference_run_is_reproduced_by_series_replay(ref, restate, prof):
    """The reference simulator's own controllers (greenllm policy, sinusoid decode load,
    acceptance check 6 shape) are replayed from their captured inputs bit-exactly."""
    a, p, o = ref.gen_sinusoid_decode_trace(1500.0, 1000.0, 120000.0, 60000, 11)
    r = ref.run_capture(a, p, o, prof, "greenllm")
    cfg = default_ctl_cfg()
    lo, hi, fo, fe = restate.band_table(prof, LEVELS, cfg.tslo_ms * cfg.margin_decode)
    tb = band_table(lo, hi, fo)
    dec = r["decisions"]
    for w in range(4):
        m, mc = r["fine_worker"] == w, r["coarse_worker"] == w
        got = restate.replay_series(cfg, tb, 210.0, 1410.0, w, r["fine_has"][m], r["fine_p95"][m],
                                    r["coarse_tps"][mc], r["fine_t"][m][-1])
        assert (got == dec[dec["worker"] == w]).all()
