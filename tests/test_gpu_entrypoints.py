"""GPU parity of the single-call / batched entry points behind the C++ drop-in
(include/gsb.h: gsb_decode_script with resumable gsb_ctl_state, gsb_quantile_batch,
gsb_tps_window_batch, gsb_steady_state_batch, gsb_classify, gsb_t_ref_batches,
gsb_energy_closed_form_batches) against the unmodified reference (oracle/_ref). Bit-exact."""
import numpy as np
import pytest
import torch

from oracle.oracle import Profile, band_table, default_ctl_cfg

pytestmark = pytest.mark.gpu

KIND_FINE, KIND_COARSE, KIND_ADAPT = 0, 1, 2


def _api():
    from paper_2508_16449_b200 import api
    return api


def u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _tables(api, ref):
    """(lo, hi, f) tables: one bucket, two buckets, the default-profile 15-level table."""
    inf = np.inf
    out = [(np.array([0.0]), np.array([inf]), np.array([705.0])),
           (np.array([0.0, 500.0]), np.array([500.0, inf]), np.array([300.0, 600.0])),
           (np.array([0.0]), np.array([inf]), np.array([1410.0])),
           (np.array([0.0]), np.array([inf]), np.array([210.0]))]
    lo, hi, fo, _ = ref.band_table(ref.default_profile(), np.arange(200.0, 3001.0, 200.0), 95.0)
    out.append((lo, hi, fo))
    return out


def _random_script(rng, n_ev, tps_max):
    kind = rng.choice([KIND_FINE] * 8 + [KIND_COARSE] * 2 + [KIND_ADAPT], size=n_ev).astype(np.int8)
    t = np.cumsum(rng.integers(0, 3, size=n_ev) * 10.0)  # non-decreasing, with repeats
    value = np.where(kind == KIND_COARSE, rng.uniform(0.0, tps_max, n_ev),
                     rng.choice([rng.uniform(5.0, 200.0), 100.0, 65.0, 95.0, 61.75], n_ev))
    value = np.where(kind == KIND_FINE, rng.uniform(5.0, 200.0, n_ev), value)
    # exact threshold hits: margin == upper / lower (p95 = margin * tslo * mult)
    edge = rng.random(n_ev) < 0.1
    value = np.where(edge & (kind == KIND_FINE), rng.choice([95.0, 61.75, 100.0, 65.0], n_ev), value)
    has = (rng.random(n_ev) > 0.15).astype(np.uint8)
    return kind, t, value, has


def _cfgs(rng, n):
    out = []
    for _ in range(n):
        kw = dict(margin_decode=float(rng.choice([0.95, 1.0, 0.5, 1.7])),
                  hysteresis_count=int(rng.integers(1, 5)),
                  bias_threshold=float(rng.choice([0.8, 0.5, 0.3, 0.95])),
                  tps_scale=float(rng.choice([1.0, 4.0, 2.5])),
                  step_mhz=float(rng.choice([15.0, 30.0])),
                  max_step_mhz=30.0,
                  lower_margin=float(rng.choice([0.65, 0.5, 0.9])))
        out.append(kw)
    return out


def _script_batch(api, ref, seed, n_ctl=96, n_ev=300):
    rng = np.random.default_rng(seed)
    tables = _tables(api, ref)
    cfg_kw = _cfgs(rng, n_ctl)
    table_of = rng.integers(0, len(tables), n_ctl).astype(np.int32)
    NB = max(len(t[0]) for t in tables)
    # pad tables to a common bucket count is not allowed (the last bucket must reach +inf), so
    # group controllers by table shape: use the shape of the largest group per launch instead
    scripts = [_random_script(rng, n_ev, 1500.0) for _ in range(n_ctl)]
    return tables, cfg_kw, table_of, NB, scripts


def _run_gpu(eng, api, tables, cfg_kw, table_of, scripts, chunks=1):
    """Run each table group through gsb_decode_script; chunks > 1 resumes from the state."""
    grid = api.FrequencyGrid()
    results = {}
    for tb in np.unique(table_of):
        idx = np.nonzero(table_of == tb)[0]
        lo, hi, fo = tables[tb]
        cfgs = [api.DecodeCtlConfig(**cfg_kw[i]) for i in idx]
        n = len(idx)
        state = None
        recs = [[] for _ in range(n)]
        n_ev = len(scripts[idx[0]][0])
        bounds = np.linspace(0, n_ev, chunks + 1).astype(int)
        for c in range(chunks):
            a, b = bounds[c], bounds[c + 1]
            ev_off = np.arange(n + 1, dtype=np.int64) * (b - a)
            cat = lambda k: np.concatenate([scripts[i][k][a:b] for i in idx])
            out = eng.decode_script(cfgs, np.zeros(n, np.int32), np.arange(n, dtype=np.int32) + 7,
                                    hi[None, :], fo[None, :], grid, ev_off, cat(0), cat(1), cat(2),
                                    cat(3), state=state, rec_cap=max(1, b - a))
            state = out["state"]
            nrec = out["n_rec"].cpu().numpy()
            slab = out["records"].cpu().numpy()
            for j in range(n):
                recs[j].append(slab[j, :nrec[j]].reshape(-1).view(api.DECISION_DTYPE))
        st = state.cpu().numpy().view(np.uint8)
        for j, i in enumerate(idx):
            s = np.frombuffer(st[j].tobytes(), dtype=np.uint8)
            import ctypes as C
            cs = api.L.CCtlState.from_buffer_copy(s.tobytes())
            results[i] = (np.concatenate(recs[j]), cs.set_point, cs.current_bucket,
                          np.array(cs.f_opt[:len(fo)]))
    return results


def _check_against_ref(api, ref, tables, cfg_kw, table_of, scripts, results):
    prof = ref.default_profile()
    for i in range(len(scripts)):
        lo, hi, fo = tables[table_of[i]]
        cfg = default_ctl_cfg(**cfg_kw[i])
        tb = band_table(lo, hi, fo)
        local = int(np.sum(table_of[:i] == table_of[i]))
        r_rec, r_cmd, r_bucket, r_fopt = ref.decode_script(cfg, tb, prof, local + 7, *scripts[i])
        g_rec, g_cmd, g_bucket, g_fopt = results[i]
        assert len(g_rec) == len(r_rec), i
        for f in ("tick_ms", "tps", "p95_tbt_ms", "band_lo", "band_hi", "command_mhz"):
            assert np.array_equal(u64(g_rec[f]), u64(r_rec[f])), (i, f)
        for f in ("worker", "bucket", "action"):
            assert np.array_equal(g_rec[f], r_rec[f]), (i, f)
        assert g_cmd == r_cmd and g_bucket == r_bucket, i
        assert np.array_equal(u64(g_fopt), u64(r_fopt)), i


def test_decode_script_matches_reference(gsb, ref):
    api = _api()
    tables, cfg_kw, table_of, _, scripts = _script_batch(api, ref, seed=11)
    res = _run_gpu(gsb, api, tables, cfg_kw, table_of, scripts, chunks=1)
    _check_against_ref(api, ref, tables, cfg_kw, table_of, scripts, res)


def test_decode_script_resumed_state_equals_one_shot(gsb, ref):
    """A controller stepped call by call through gsb_ctl_state (how the C++ DecodeController
    drives the kernel) produces the reference's log exactly, chunk size notwithstanding."""
    api = _api()
    tables, cfg_kw, table_of, _, scripts = _script_batch(api, ref, seed=12, n_ctl=40, n_ev=120)
    for chunks in (7, 120):
        res = _run_gpu(gsb, api, tables, cfg_kw, table_of, scripts, chunks=chunks)
        _check_against_ref(api, ref, tables, cfg_kw, table_of, scripts, res)


def test_quantile_batch_matches_reference(gsb, ref):
    rng = np.random.default_rng(5)
    # > 4096 samples: the radix-select path (the reference takes any size; io.cpp's tbt_digest
    # feeds it a request's whole TBT list)
    sizes = np.concatenate([[1, 2, 3, 4, 5, 19, 20, 21, 255, 256, 257, 1024, 4095, 4096, 4097,
                             9000, 70_001, 300_000], rng.integers(1, 4097, 30)])
    sets = []
    for n in sizes:
        kind = rng.integers(0, 3)
        if kind == 0:
            s = rng.uniform(0, 200, n)
        elif kind == 1:
            s = rng.integers(0, 7, n).astype(np.float64)  # heavy ties
        else:
            s = np.concatenate([rng.normal(50, 10, n - n // 3), np.full(n // 3, -0.0),
                                ])[:n]
        sets.append(s)
    off = np.concatenate([[0], np.cumsum([len(s) for s in sets])]).astype(np.int64)
    flat = np.concatenate(sets)
    for q in (0.0, 0.5, 0.95, 0.99, 1.0, 0.123456789):
        got = gsb.quantile_batch(off, flat, q).cpu().numpy()
        want = np.array([ref.quantile(s, q) for s in sets])
        assert np.array_equal(u64(got), u64(want)), q


def test_tps_window_batch_matches_reference(gsb, ref):
    rng = np.random.default_rng(6)
    offs, ts, ks, ws, nows, want = [0], [], [], [], [], []
    for w in range(500):
        n = int(rng.integers(0, 60))
        t = np.sort(rng.integers(0, 2000, n).astype(np.float64) + rng.choice([0.0, 0.5], n))
        k = rng.integers(0, 64, n).astype(np.int32)
        win = float(rng.choice([200.0, 100.0, 37.5]))
        now = float(rng.choice([t[-1] if n else 0.0, 1000.0, 2000.0, (t[n // 2] + win) if n else 5.0]))
        ts.append(t), ks.append(k), ws.append(win), nows.append(now)
        offs.append(offs[-1] + n)
        want.append(ref.tps_window(win, t, k, now))
    got = gsb.tps_window_batch(np.array(offs, np.int64), np.concatenate(ts), np.concatenate(ks),
                               np.array(ws), np.array(nows)).cpu().numpy()
    assert np.array_equal(u64(got), u64(np.array(want)))


def test_steady_state_batch_matches_reference(gsb, ref):
    api = _api()
    prof = ref.default_profile()
    p = api.GpuProfile.default_profile()
    rng = np.random.default_rng(8)
    grid = np.arange(210.0, 1410.0 + 1e-9, 15.0)
    tps = np.concatenate([rng.uniform(0, 4000, 3000), [0.0, 1.0, 1e-9, 2719.9, 1e6]])
    f = rng.choice(grid, len(tps))
    mb = rng.choice([1, 8, 64, 256], len(tps)).astype(np.int32)
    sus, b, t = (x.cpu().numpy() for x in gsb.steady_state_batch(p, tps, f, mb))
    for i in range(len(tps)):
        rs, rb, rt = ref.steady_state(prof, tps[i], f[i], int(mb[i]))
        assert bool(sus[i]) == bool(rs), i
        assert u64([b[i]])[0] == u64([rb])[0] and u64([t[i]])[0] == u64([rt])[0], i


def test_classify_matches_reference(gsb, ref):
    api = _api()
    rng = np.random.default_rng(9)
    prompts = np.concatenate([rng.integers(-5, 70000, 20000), [0, 1, 1024, 1025, 2**31 - 1]])
    for thr in ([1024], [256, 1024, 4096], [4096, 256], [1, 2, 3, 4, 5, 6, 7], [7, 7]):
        rc = api.RoutingConfig(thresholds=list(thr), worker_map=list(range(len(thr) + 1)))
        got = gsb.classify_many(rc, prompts)
        want = np.array([ref.classify(thr, int(x)) for x in prompts[::37]])
        assert np.array_equal(got[::37], want), thr


def test_t_ref_and_closed_form_match_reference(gsb, ref):
    api = _api()
    rng = np.random.default_rng(10)
    prof = ref.default_profile()
    p = api.GpuProfile.default_profile()
    n_b = 400
    sizes = rng.integers(0, 9, n_b)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    prompts = rng.integers(1, 9000, off[-1]).astype(np.int32)
    wf = rng.uniform(0.0, 1.0, off[-1])
    lat = api.LatencyModel(p.prefill.a, p.prefill.b, p.prefill.c, 1410.0)
    t = gsb.t_ref_batches(lat, off, prompts, wf).cpu().numpy()
    f = rng.choice(np.arange(210.0, 1411.0, 15.0), n_b)
    f[::17] = 211.0  # off grid -> NaN (the reference throws)
    W = rng.uniform(10, 5000, n_b)
    cf = gsb.energy_closed_form_batches(off, prompts, f, W, p, wf).cpu().numpy()
    for b in range(n_b):
        pr, w = prompts[off[b]:off[b + 1]], wf[off[b]:off[b + 1]]
        assert u64([t[b]])[0] == u64([ref.t_ref(prof, pr, w)])[0], b
        if f[b] == 211.0:
            assert np.isnan(cf[b])
        else:
            assert u64([cf[b]])[0] == u64([ref.closed_form(prof, pr, f[b], W[b], w)])[0], b


def test_unchecked_profiles_evaluate_like_the_reference(gsb, ref):
    """Flat / non-monotone power (rejected by validate(), accepted by the reference's
    evaluators, test_prefill_opt.cpp:98,135) through gsb_set_profiles_ex(UNCHECKED)."""
    import ctypes as C
    api = _api()
    L = api.L
    rng = np.random.default_rng(13)
    for k3, k2, k1, k0, idle in [(0, 0, 0, 80.0, 1e-9), (0, 0, -0.01, 90.0, 5.0),
                                 (1e-9, 0.0, 0.1, 50.0, 60.0)]:
        p = api.GpuProfile.default_profile()
        p.power = api.PowerModel(k3, k2, k1, k0, idle)
        c = p.to_c()
        assert gsb.lib.gsb_set_profiles(gsb.ctx, 1, C.byref(c)) in (L.OK, L.MODEL_ERROR)
        assert gsb.lib.gsb_set_profiles_ex(gsb.ctx, 1, C.byref(c), 1) == L.OK
        gsb.profiles = [p]
        rp = Profile(*p.key())
        sizes = rng.integers(1, 5, 200)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        prompts = rng.integers(16, 4096, off[-1]).astype(np.int32)
        W = rng.uniform(10, 4000, 200)
        f_idx, e, _, _ = gsb.select_batches(off, prompts, W, None)
        f_idx, e = f_idx.cpu().numpy(), e.cpu().numpy()
        for b in range(200):
            r = ref.select_frequency(rp, prompts[off[b]:off[b + 1]], W[b])
            if r is None:
                assert f_idx[b] == -1
            else:
                assert p.grid.at(int(f_idx[b])) == r[0] and u64([e[b]])[0] == u64([r[1]])[0], b
    gsb.set_profiles([api.GpuProfile.default_profile()])


def test_mg1_side_output_formula(gsb):
    """North_star (2)'s M/G/1 side output: PARITY-UNPINNED (the reference has no M/G/1 term,
    SPEC.md:294), so it is pinned to its own definition (Pollaczek-Khinchine over the cell's
    service times at the command's clock), computed here in float64 numpy, 1e-12 relative."""
    import torch
    from paper_2508_16449_b200 import api, workloads as wl
    profs = wl.synth_profiles(2)
    gsb.set_profiles(profs)
    a, p, _ = wl.poisson_trace(5.0, 120 * 60_000, "alibaba_chat", seed=9)
    routing = api.RoutingConfig(True, wl.THRESHOLDS[3], [0, 1, 2])
    rr = gsb.route_bin(a, p, routing, 60_000, 0, 120)
    sel = gsb.prefill_select(rr, api.L.FIXED_WINDOW, fixed_window_ms=57_000.0)
    out = gsb.mg1_side_output(rr, sel, p)
    torch.cuda.synchronize()
    cls = rr.cls.cpu().numpy()
    fi, en = sel.f_idx.cpu().numpy(), sel.energy_j.cpu().numpy()
    wq, rho, epr = (out[k].cpu().numpy() for k in ("wq_ms", "rho", "energy_per_request_j"))
    win = a // 60_000
    checked = 0
    for pi, pr in enumerate(profs):
        grid = np.array(pr.grid.frequencies())
        for cell in range(0, 360, 7):
            w, c = divmod(cell, 3)
            m = (win == w) & (cls == c)
            if fi[pi, cell] == -2:
                assert m.sum() == 0 and wq[pi, cell] == 0.0
                continue
            L = p[m].astype(np.float64)
            t = (pr.prefill.a * L + pr.prefill.b) * L + pr.prefill.c
            f = grid[fi[pi, cell]] if fi[pi, cell] >= 0 else pr.grid.f_max_mhz
            k = pr.grid.f_ref_mhz / f
            lam = len(L) / 60_000.0
            r = lam * k * t.sum() / len(L)
            assert abs(rho[pi, cell] - r) <= 1e-12 * r
            want = lam * k * k * (t * t).sum() / len(L) / (2 * (1 - r)) if r < 1 else np.inf
            assert (wq[pi, cell] == want) if not np.isfinite(want) else abs(wq[pi, cell] - want) <= 1e-12 * want
            if fi[pi, cell] >= 0:
                assert abs(epr[pi, cell] - en[pi, cell] / len(L)) <= 1e-15 * en[pi, cell]
            checked += 1
    assert checked > 50
