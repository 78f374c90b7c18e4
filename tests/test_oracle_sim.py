"""Pins the restated simulator (oracle/gs_sim.c) against the reference's own run()
(proj/src/simkernel.cpp), field by field and bit for bit, and shows that the decode pool
replayed from one recorded enqueue stream reproduces the reference's decode-side outputs at
other controller parameters (the property K5 relies on)."""
import numpy as np
import pytest

from oracle.oracle import (PolicyHolder, default_ctl_cfg, default_qopt_cfg, default_sim_cfg,
                           default_slo)

SKIP = {"n_steps", "scalars", "enq_t", "enq_req", "summary"}


def _same(ref_out, our):
    for k, x in ref_out.items():
        if k in SKIP:
            continue
        y = our[k]
        if isinstance(x, np.ndarray):
            assert x.shape == y.shape and x.tobytes() == y.tobytes(), k
        else:
            assert x == y, k


@pytest.fixture(scope="module")
def sinus(ref):
    return ref.gen_sinusoid_decode_trace(1500.0, 1000.0, 120000.0, 150000, 11)


@pytest.fixture(scope="module")
def poisson(ref):
    # Alibaba-chat-shaped, 10 minutes
    return ref.gen_poisson_trace(5.0, 600_000, 512.0, 4096.0, 0.10, 128.0, 7)


CASES = {
    "greenllm_default": dict(),
    "greenllm_3class": dict(policy=dict(thresholds=(512, 1024), worker_map=(0, 1, 2)),
                            cfg=dict(n_prefill_workers=3)),
    "defaultnv": dict(policy=dict(kind="defaultnv", routing=False)),
    "fixed_900": dict(policy=dict(kind="fixed", fixed_f=900.0, routing=False)),
    "prefillsplit": dict(policy=dict(kind="prefillsplit")),
    "overload": dict(cfg=dict(max_batch=4, max_queue=6, n_decode_workers=2)),
    "handoff_delay": dict(cfg=dict(handoff_delay_ms=7.5, actuation_delay_ms=12.0)),
    "tight_slo": dict(slo=dict(tbt_p95_ms=60.0, ttft_sm_ms=150.0),
                      policy=dict(ccfg=dict(tslo_ms=60.0, hysteresis_count=1))),
}


def _build(case, prof):
    c = CASES[case]
    pk = dict(c.get("policy", {}))
    ccfg = default_ctl_cfg(**pk.pop("ccfg", {}))
    pol = PolicyHolder(ccfg=ccfg, qcfg=default_qopt_cfg(), **pk)
    return pol, default_slo(**c.get("slo", {})), default_sim_cfg(**c.get("cfg", {}))


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("trace", ["sinus", "poisson"])
def test_restated_sim_equals_reference_run(ref, restate, prof, sinus, poisson, case, trace):
    a, p, o = sinus if trace == "sinus" else poisson
    pol, slo, cfg = _build(case, prof)
    r = ref.sim_run(prof, pol, slo, cfg, a, p, o)
    g = restate.sim_run(prof, pol, slo, cfg, a, p, o)
    _same(r, g)
    assert r["scalars"][0] == g["scalars"][0]  # sim_end_ms
    # the K5 summary computed from the reference's RunResult equals the restatement's
    s_ref = restate.pool_summary_from(slo, a.astype(np.float64), r)
    s_our = g["summary"]
    for k in s_ref:
        if k != "n_steps":
            assert s_ref[k] == s_our[k], k
    # and its pass counts reproduce the reference's own slo_pass_rates (metrics.cpp:42-72)
    n = s_our["n_completed"]
    if n:
        assert 100.0 * s_our["n_ttft_ok"] / n == r["scalars"][5]
        assert 100.0 * s_our["n_tbt_ok"] / n == r["scalars"][6]
        ts = s_our["tbt_samples"]
        agg = 100.0 if ts == 0 else 100.0 * s_our["tbt_samples_ok"] / ts
        assert agg == r["scalars"][7]
    if case == "overload":
        assert s_our["n_rejected"] > 0 or g["n_rejected_total"] > 0


VARIANTS = [dict(), dict(hysteresis_count=1), dict(hysteresis_count=5),
            dict(step_mhz=30.0, max_step_mhz=30.0), dict(step_mhz=15.0, max_step_mhz=45.0),
            dict(margin_decode=0.6), dict(margin_decode=1.5, upper_margin=0.9, lower_margin=0.5),
            dict(tslo_ms=60.0), dict(adapt_period_s=2.0, bias_threshold=0.5),
            dict(tbt_window_tokens=32), dict(fine_period_ms=25.0, coarse_period_ms=150.0)]


@pytest.mark.parametrize("kw", VARIANTS, ids=[str(v) for v in VARIANTS])
def test_stream_replay_equals_reference_at_other_parameters(ref, restate, prof, sinus, kw):
    """One stream recorded at the default parameters drives every variant: the decode-side
    outputs of gso_pool_run equal the reference's full run() at that variant."""
    a, p, o = sinus
    pol0, slo, cfg = _build("greenllm_default", prof)
    g0 = restate.sim_run(prof, pol0, slo, cfg, a, p, o)
    pol = PolicyHolder(ccfg=default_ctl_cfg(**kw))
    r = ref.sim_run(prof, pol, slo, cfg, a, p, o)
    q = restate.pool_run(prof, pol, slo, cfg, a, p, o, g0["enq_t"], g0["enq_req"],
                         g0["scalars"][2])
    s_ref = restate.pool_summary_from(slo, a.astype(np.float64), r)
    for k in s_ref:
        if k != "n_steps":
            assert s_ref[k] == q["summary"][k], k
    assert r["decisions"].tobytes() == q["decisions"].tobytes()
    assert r["tbt"].tobytes() == q["tbt"].tobytes()
    assert r["decode3"].tobytes() == q["decode3"].tobytes()


def test_enqueue_stream_is_parameter_independent(restate, prof, sinus):
    a, p, o = sinus
    pol0, slo, cfg = _build("greenllm_default", prof)
    g0 = restate.sim_run(prof, pol0, slo, cfg, a, p, o)
    for kw in (dict(hysteresis_count=1), dict(margin_decode=1.5)):
        g = restate.sim_run(prof, PolicyHolder(ccfg=default_ctl_cfg(**kw)), slo, cfg, a, p, o)
        assert g["enq_t"].tobytes() == g0["enq_t"].tobytes()
        assert g["enq_req"].tobytes() == g0["enq_req"].tobytes()
        assert g["scalars"][2] == g0["scalars"][2]


def test_restated_snapshots_match_reference_capture(restate, ref, prof):
    """The restated simulator's optimizer snapshots (with the raw running-job state the device
    work_fraction test replays) are the reference simulator's own: same queues, prompts,
    deadlines and work_fraction bits (simkernel.cpp:466-501)."""
    from oracle import oracle as O
    a, p, o = ref.gen_poisson_trace(5.0, 1_200_000, seed=7)
    r = ref.run_capture(a, p, o, prof, "greenllm", thresholds=(512, 1024), worker_map=(0, 1, 2))
    pol = O.PolicyHolder("greenllm", thresholds=(512, 1024), worker_map=(0, 1, 2))
    sn = restate.sim_run(prof, pol, O.default_slo(), O.default_sim_cfg(n_prefill_workers=3),
                         a, p, o)["snapshots"]
    off = r["snap_off"]
    idx = np.nonzero(np.diff(off) > 0)[0]
    sel = np.concatenate([np.arange(off[i], off[i + 1]) for i in idx])
    np.testing.assert_array_equal(sn["now"], r["snap_now"][idx])
    np.testing.assert_array_equal(sn["cls"], r["snap_class"][idx])
    np.testing.assert_array_equal(sn["prompt"], r["job_prompt"][sel])
    np.testing.assert_array_equal(sn["deadline"].view(np.uint64), r["job_deadline"][sel].view(np.uint64))
    np.testing.assert_array_equal(sn["wf"].view(np.uint64), r["job_wf"][sel].view(np.uint64))
    # the raw state reproduces the fraction in the reference's operation order
    run = sn["running"] != 0
    done = (np.repeat(sn["now"], np.diff(sn["off"]))[run] - sn["upd_ms"][run]) * sn["freq"][run] / 1410.0
    wf = np.maximum(sn["rem_ref"][run] - done, 0.0) / sn["t_ref"][run]
    np.testing.assert_array_equal(wf.view(np.uint64), sn["wf"][run].view(np.uint64))
    assert run.sum() > 1000
