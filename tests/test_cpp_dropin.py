"""The C++ drop-in boundary ("Existing C++ API must stay unchanged").

The reference's own unit tests for the path — proj/tests/test_prefill_opt.cpp,
test_decode_ctl.cpp, test_router.cpp — plus test_simkernel.cpp (the reference simulator's tests,
whose governed runs take every routing / clock / controller decision through the drop-in) are
compiled UNMODIFIED against paper_2508_16449_b200/cpp/include (greensim/*.hpp) and linked to
libgreensim_b200.so -> libgsb.so (build: paper_2508_16449_b200/cpp/Makefile, into
oracle/_ref/dropin/). On a B200 every case must pass with every evaluation running in the sm_100a
kernels; without a GPU the binaries must refuse (no CPU path).
"""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2508_16449_b200", "lib")
# the reference's own unit tests, unmodified; test_router / test_simkernel run the reference's
# simulator compiled over the drop-in (every decision it takes is a libgsb launch)
REF_BINS = [os.path.join(ROOT, "oracle", "_ref", "dropin", n)
            for n in ("test_prefill_opt", "test_decode_ctl", "test_router", "test_simkernel")]
OWN_BINS = [os.path.join(ROOT, "tests", "cpp", "bin", n)
            for n in ("test_router_dropin", "test_acceptance_dropin", "test_trace_dropin")]
ALL_BINS = REF_BINS + OWN_BINS


def _run(path: str, timeout: int = 600) -> subprocess.CompletedProcess:
    return subprocess.run([path], capture_output=True, text=True, timeout=timeout)


def test_dropin_library_exports_reference_api():
    """libgreensim_b200.so defines the reference's greensim:: entry points (mangled C++ names)."""
    so = os.path.join(LIB, "libgreensim_b200.so")
    assert os.path.exists(so), "build the C++ drop-in first (__graft_entry__.build())"
    out = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True, text=True,
                         check=True).stdout
    for sym in ["greensim::select_frequency(", "greensim::queue_optimizer_tick(",
                "greensim::energy_total(", "greensim::busy_time_ms(",
                "greensim::PrefillBatch::t_ref_total_ms(", "greensim::classify(",
                "greensim::Dispatcher::dispatch(", "greensim::build_band_table(",
                "greensim::decode_steady_state(", "greensim::DecodeController::on_fine_tick(",
                "greensim::DecodeController::on_coarse_tick(",
                "greensim::DecodeController::on_adapt_tick(", "greensim::audit_decision_log(",
                "greensim::decision_log_csv", "greensim::TbtWindow::p95()",
                "greensim::TpsWindow::tps(", "greensim::quantile(", "greensim::load_trace(",
                "greensim::save_trace_csv("]:
        assert sym in out, sym
    # and it is a client of the C ABI, not a second implementation
    dyn = subprocess.run(["nm", "-D", "--undefined-only", so], capture_output=True, text=True,
                         check=True).stdout
    for sym in ["gsb_select_batches", "gsb_decode_script", "gsb_build_band_tables", "gsb_classify",
                "gsb_trace_parse", "gsb_trace_format"]:
        assert sym in dyn, sym


@pytest.mark.parametrize("path", ALL_BINS, ids=os.path.basename)
def test_dropin_refuses_without_gpu(path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu-marked run")
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (reference tests need /root/reference at build time)")
    r = _run(path, timeout=120)
    assert r.returncode != 0
    assert "no CPU path" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("path", ALL_BINS, ids=os.path.basename)
def test_dropin_unit_tests_pass_on_b200(path):
    assert os.path.exists(path), f"{path} missing: run __graft_entry__.build() where /root/reference exists"
    r = _run(path)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed" in r.stdout
