"""CPU-side checks of the drop-in boundary: libgsb.so loads, exports every function
include/gsb.h declares, refuses to run without a B200 (no silent CPU path), and its
host-side validators agree with the reference's typed-exception rules."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from oracle.oracle import CtlCfg, Profile, default_ctl_cfg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build_lib()
    from paper_2508_16449_b200 import _lib
    return _lib.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "gsb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gsb_[a-z0-9_]+)\s*\(", src)))


def test_header_and_exports_agree(lib):
    from paper_2508_16449_b200 import _lib
    declared = header_functions()
    assert set(declared) == set(_lib.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (gsb_[a-z0-9_]+)", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    for f in declared:
        getattr(lib, f)  # resolvable through ctypes


def test_library_is_sm100a_only(lib):
    from paper_2508_16449_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_gpu_means_loud_failure(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    assert lib.gsb_ctx_create(0, C.byref(h)) == 4  # GSB_CUDA_ERROR, never a CPU fallback
    from paper_2508_16449_b200 import api
    with pytest.raises(Exception):
        api.Engine(0)


def _cprof(p):
    from paper_2508_16449_b200 import _lib
    return _lib.CProfile(*p.tuple())


def test_profile_validation_matches_reference(lib, ref, prof):
    rng = np.random.default_rng(4)
    msg = C.create_string_buffer(256)
    fields = [n for n, _ in Profile._fields_]
    for it in range(400):
        p = Profile(*prof.tuple())
        k = fields[it % len(fields)]
        v = getattr(p, k)
        setattr(p, k, v * rng.choice([-1.0, 0.0, 0.5, 1.0000000001, 3.0]))
        mine = lib.gsb_profile_validate(C.byref(_cprof(p)), msg, 256)
        if b"GSB_MAX_GRID" in msg.value:
            continue  # documented capacity limit of the kernels, not a reference rule
        assert (mine == 0) == ref.validate(p), (k, getattr(p, k), msg.value)
        if mine:
            assert mine == 1  # GSB_MODEL_ERROR


def test_ctl_cfg_validation_matches_reference(lib, ref):
    from paper_2508_16449_b200 import _lib
    base = default_ctl_cfg()
    fields = [n for n, _ in CtlCfg._fields_]
    msg = C.create_string_buffer(256)
    for k in fields:
        for mul in (-1.0, 0.0, 0.1, 0.5, 1.0, 2.5):
            c = default_ctl_cfg()
            v = getattr(base, k)
            setattr(c, k, type(v)(v * mul))
            cc = _lib.CCtlCfg(*[getattr(c, f) for f in fields])
            mine = lib.gsb_ctl_cfg_validate(C.byref(cc), msg, 256)
            want = ref.lib.ref_ctl_cfg_validate(C.byref(c))
            assert (mine == 0) == (want == 0), (k, mul, msg.value)


def test_routing_validation(lib):
    from paper_2508_16449_b200 import api
    api.RoutingConfig(True, [1024], [0, 1]).validate(2)
    for thr, wm, n in (([1024, 1024], [0, 1], 2), ([2048, 1024], [0, 1], 2), ([1024], [0, 0], 2),
                       ([1024], [0, 1, 1], 2), ([0], [0, 1], 2), ([], [0], 1)):
        with pytest.raises(api.RouterError):
            api.RoutingConfig(True, thr, wm).validate(n)
    api.RoutingConfig(False, [1024], []).validate(2)


def test_tick_count_matches_oracle(lib, restate):
    for period, t_end in ((20.0, 150_000.0), (200.0, 150_000.0), (6000.0, 150_000.0),
                          (0.1, 100.0), (7.3, 1234.5)):
        assert lib.gsb_n_ticks(period, t_end) == restate.n_ticks(period, t_end)
