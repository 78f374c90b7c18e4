"""N > 1 host logic on CPU: window sharding, the gloo all-gather of per-class summaries and
the rank-order combine, checked against a single-process pass over all windows (the
per-cell decisions come from the CPU oracle here; on the GPU they come from K1/K2)."""
import os
import socket

import numpy as np
import pytest

from paper_2508_16449_b200 import distributed as D

THR = [512, 1024]
WMS = 5_000
TOTAL_W = 157


def _summary(fi, en, C):
    """numpy restatement of gsb_prefill_summary for one profile: [C] SUMMARY_DTYPE."""
    out = np.zeros(C, D.SUMMARY_DTYPE)
    fi = fi.reshape(-1, C)
    en = en.reshape(-1, C)
    for c in range(C):
        f, e = fi[:, c], en[:, c]
        out[c]["n_empty"] = (f == -2).sum()
        out[c]["n_cmd"] = (f != -2).sum()
        out[c]["n_infeasible"] = (f == -1).sum()
        ok = f >= 0
        out[c]["sum_energy_j"] = float(np.sum(e[ok]))
        if ok.any():
            k = int(np.argmin(np.where(ok, e, np.inf)))
            out[c]["min_energy_j"] = e[k]
            out[c]["argmin_cell"] = k * C + c
        else:
            out[c]["min_energy_j"] = np.inf
            out[c]["argmin_cell"] = -1
    return out


def _decide(restate, prof, a, p, w0, n):
    cls, cnt, tref, mdl, _ = restate.route_bin(a, p, THR, WMS, w0, n, [prof], fifo=False)
    C = len(THR) + 1
    fi = np.full(n * C, -2, np.int64)
    en = np.zeros(n * C)
    for cell in range(n * C):
        if cnt[cell]:
            r = restate.select_t(prof, tref[0, cell], 0.95 * WMS)
            fi[cell], en[cell] = (-1, 0.0) if r is None else (r[0], r[2])
    return fi, en


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from oracle.oracle import Restatement, default_profile
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    R = Restatement()
    prof = default_profile()
    a, p, _ = R.gen_poisson_trace(6.0, TOTAL_W * WMS, seed=5)
    w0, n = D.window_shard(TOTAL_W, world, rank)
    lo, hi = D.trace_slice(a, WMS, w0, n)
    fi, en = _decide(R, prof, a[lo:hi], p[lo:hi], w0, n)
    s = _summary(fi, en, len(THR) + 1)
    t = torch.from_numpy(s.view(np.uint8).reshape(len(THR) + 1, -1).copy())
    g = D.gather_summaries(t)
    per_rank = g.numpy().reshape(world, -1).view(D.SUMMARY_DTYPE).reshape(world, 1, -1)
    offsets = [D.window_shard(TOTAL_W, world, r)[0] * (len(THR) + 1) for r in range(world)]
    comb = D.combine_summaries(per_rank, offsets)
    np.save(os.path.join(out_dir, f"comb{rank}.npy"), comb)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_window_shard_covers_everything():
    for total in (1, 7, 100, 10_001):
        for world in (1, 2, 3, 8):
            got = [D.window_shard(total, world, r) for r in range(world)]
            assert got[0][0] == 0
            for (w0, n), (w1, _) in zip(got, got[1:]):
                assert w0 + n == w1
            assert sum(n for _, n in got) == total


def test_trace_slice_matches_window_rule(restate):
    a, _, _ = restate.gen_poisson_trace(3.0, 10 * WMS, seed=1)
    for w0, n in ((0, 3), (2, 5), (9, 1), (0, 10)):
        lo, hi = D.trace_slice(a, WMS, w0, n)
        w = a // WMS
        assert np.all((w[lo:hi] >= w0) & (w[lo:hi] < w0 + n))
        assert lo == 0 or w[lo - 1] < w0
        assert hi == len(a) or w[hi] >= w0 + n


def test_two_rank_gloo_combine_matches_single_pass(restate, prof, tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    c0 = np.load(tmp_path / "comb0.npy")
    c1 = np.load(tmp_path / "comb1.npy")
    assert c0.tobytes() == c1.tobytes()  # bitwise identical on every rank
    a, p, _ = restate.gen_poisson_trace(6.0, TOTAL_W * WMS, seed=5)
    fi, en = _decide(restate, prof, a, p, 0, TOTAL_W)
    single = _summary(fi, en, len(THR) + 1)
    comb = c0[0]
    for k in ("n_cmd", "n_infeasible", "n_empty", "argmin_cell", "min_energy_j"):
        np.testing.assert_array_equal(comb[k], single[k])
    np.testing.assert_allclose(comb["sum_energy_j"], single["sum_energy_j"], rtol=1e-9)
    assert comb["n_infeasible"].sum() > 0 and comb["n_empty"].sum() >= 0


def _pool_records(n, seed):
    """Synthetic per-scenario gsb_pool_summary records (the K5 output format)."""
    from paper_2508_16449_b200.api import POOL_SUMMARY_DTYPE
    rng = np.random.default_rng(seed)
    sm = np.zeros(n, POOL_SUMMARY_DTYPE)
    sm["decode_pool_j"] = rng.uniform(1e5, 2e5, n)
    for k in ("n_completed", "n_rejected", "n_ttft_ok", "n_tbt_ok", "tbt_samples",
              "tbt_samples_ok", "n_decisions", "n_freq_changes"):
        sm[k] = rng.integers(0, 10_000, n)
    for k in ("decision_digest", "freq_digest", "request_digest"):
        sm[k] = rng.integers(0, 2**63, n, dtype=np.int64).astype(np.uint64)
    sm["decode_pool_j"][n // 3] = 50_000.0  # a unique minimum
    return sm


def _pool_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sm = _pool_records(1000, 3)
    lo, n = D.scenario_shard(len(sm), world, rank)
    mine = D.tally_pool(sm[lo:lo + n], lo)
    per_rank = D.gather_records(np.array([mine], D.DECODE_TALLY_DTYPE), "cpu")
    np.save(os.path.join(out_dir, f"pool{rank}.npy"), np.array([D.combine_tallies(per_rank)]))
    dist.destroy_process_group()


def test_decode_pool_tallies_gloo_world2(tmp_path):
    """Decode-side end-of-run reduction: two ranks tally their scenario
    ranges, all-gather, combine in rank order: identical bytes on both ranks; counts, digest
    and argmin equal the single-process tally exactly, energy within 1e-12."""
    import torch.multiprocessing as mp
    mp.spawn(_pool_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "pool0.npy")
    r1 = np.load(tmp_path / "pool1.npy")
    assert r0.tobytes() == r1.tobytes()
    single = D.tally_pool(_pool_records(1000, 3), 0)
    g = r0[0]
    for k in D.DECODE_TALLY_DTYPE.names:
        if k == "decode_pool_j":
            assert abs(g[k] - single[k]) <= 1e-12 * abs(single[k])
        else:
            assert g[k] == single[k], k
    assert g["argmin_scenario"] == 1000 // 3


def test_decode_tallies_split_invariance():
    """tally_pool/combine_tallies: any split of the scenarios over ranks (including empty
    ranks) gives the same counts, digest and argmin as one tally; energy within 1e-12."""
    sm = _pool_records(257, 11)
    single = D.tally_pool(sm, 0)
    for world in (1, 2, 3, 8, 300):
        parts = []
        for r in range(world):
            lo, n = D.scenario_shard(len(sm), world, r)
            parts.append(D.tally_pool(sm[lo:lo + n], lo))
        g = D.combine_tallies(np.array(parts, D.DECODE_TALLY_DTYPE))
        for k in D.DECODE_TALLY_DTYPE.names:
            if k == "decode_pool_j":
                assert abs(g[k] - single[k]) <= 1e-12 * abs(single[k])
            else:
                assert g[k] == single[k], (world, k)


def test_c_abi_reductions_equal_the_python_combine():
    """gsb_combine_summaries / gsb_tally_pool / gsb_combine_tallies (host C over the C ABI, what
    a C++ host calls after its ncclAllGather) give the Python reference combine's exact bytes."""
    rng = np.random.default_rng(6)
    R, N = 5, 24
    pr = np.zeros((R, N), D.SUMMARY_DTYPE)
    for k in ("n_cmd", "n_infeasible", "n_empty"):
        pr[k] = rng.integers(0, 1000, (R, N))
    pr["sum_energy_j"] = rng.uniform(0, 1e9, (R, N))
    pr["min_energy_j"] = rng.choice([1.0, 2.0, 3.0, np.inf], (R, N))
    pr["argmin_cell"] = np.where(np.isinf(pr["min_energy_j"]), -1, rng.integers(0, 500, (R, N)))
    off = np.arange(R) * 1000
    want = D.combine_summaries(pr.reshape(R, 1, N), off)[0]
    got = D.combine_summaries_c(pr.reshape(R, 1, N), off)[0]
    assert got.tobytes() == want.tobytes()
    sm = _pool_records(301, 2)
    assert D.tally_pool_c(sm, 17).tobytes() == D.tally_pool(sm, 17).tobytes()
    parts = np.array([D.tally_pool(sm[i::3], 100 * i) for i in range(3)], D.DECODE_TALLY_DTYPE)
    assert D.combine_tallies_c(parts).tobytes() == D.combine_tallies(parts).tobytes()


def test_host_pass_chunk_split_and_summary_combine():
    """gsb_prefill_pass_host's window chunks (decreasing sizes, weights K..1, gsb.h) cover every
    window once, and its per-chunk summary records combine like ranks (argmin cells offset by the
    chunk starts): the C combine equals the Python rank-order combine."""
    import torch
    from paper_2508_16449_b200 import api
    from paper_2508_16449_b200.distributed import SUMMARY_DTYPE, combine_summaries
    rng = np.random.default_rng(5)
    for nW, K in [(10_000, 3), (7, 7), (1440, 4), (1_000_000, 16), (5, 1)]:
        C, P = 8, 4
        r = api.HostPassResult(None, None, None, K, nW, C)
        a = r.chunk_windows()
        assert a[0] == 0 and a[-1] == nW and len(a) == K + 1
        sizes = np.diff(a)
        assert (sizes >= 0).all() and sizes.sum() == nW
        if nW >= 10 * K:
            assert (np.diff(sizes) <= 1).all()  # non-increasing (up to rounding)
        recs = np.zeros((K, P * C), SUMMARY_DTYPE)
        recs["n_cmd"] = rng.integers(0, 50, recs.shape)
        recs["n_infeasible"] = rng.integers(0, 5, recs.shape)
        recs["n_empty"] = rng.integers(0, 50, recs.shape)
        recs["sum_energy_j"] = rng.random(recs.shape) * 1e3
        recs["min_energy_j"] = rng.random(recs.shape)
        recs["argmin_cell"] = rng.integers(0, max(1, nW // K) * C, recs.shape)
        r.chunk_summaries = torch.from_numpy(recs.view(np.uint8).reshape(K, -1).copy())
        got = r.summary()
        want = combine_summaries(recs.reshape(K, P, C), [x * C for x in a[:-1]]).reshape(-1)
        assert got.tobytes() == want.tobytes()
