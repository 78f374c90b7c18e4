"""Pins the plain-C restatement of load_trace / save_trace_csv (oracle/gs_trace.c) to the
reference itself (oracle/_ref: trace.cpp compiled unmodified) and to the committed golden
fixture (tests/golden/trace_cases.json, written by tests/golden/make_trace_golden.py from the
reference)."""
import json
import os

import numpy as np
import pytest

from trace_cases import CASES, tile_straddle_case

GOLD = os.path.join(os.path.dirname(__file__), "golden", "trace_cases.json")


def _norm(r):
    if isinstance(r[0], str):
        return {"error": [r[1], r[2], r[3]]}
    return {"arrival": [int(x) for x in r[0]], "prompt": [int(x) for x in r[1]],
            "output": [int(x) for x in r[2]], "cls": [int(x) for x in r[3]]}


def test_restatement_matches_golden(restate):
    gold = json.load(open(GOLD))
    assert len(gold) == len(CASES)
    for name, data, thr in CASES:
        assert _norm(restate.trace_parse(data, thr)) == gold[name], name


@pytest.mark.parametrize("name,data,thr", CASES, ids=[c[0] for c in CASES])
def test_restatement_equals_reference_load_trace(restate, ref, tmp_path, name, data, thr):
    f = tmp_path / "t.csv"
    f.write_bytes(data)
    assert _norm(restate.trace_parse(data, thr)) == _norm(ref.load_trace(str(f), thr))


@pytest.mark.parametrize("crlf", [False, True])
def test_restatement_equals_reference_large(restate, ref, tmp_path, crlf):
    data = tile_straddle_case(5000, crlf)
    f = tmp_path / "t.csv"
    f.write_bytes(data)
    assert _norm(restate.trace_parse(data, 1024)) == _norm(ref.load_trace(str(f), 1024))


def test_writer_equals_reference_save_trace_csv(restate, ref, tmp_path):
    rng = np.random.default_rng(3)
    n = 2000
    a = np.sort(rng.integers(0, 10**12, n)).astype(np.int64)
    a[:3] = [-5, np.iinfo(np.int64).min, np.iinfo(np.int64).max]  # ostream corner values
    p = rng.integers(-(2**31), 2**31 - 1, n, dtype=np.int64).astype(np.int32)
    o = rng.integers(1, 5000, n).astype(np.int32)
    c = (p > 1024).astype(np.uint8)
    for cls in (None, c):
        got = restate.trace_format(a, p, o, cls)
        assert got == ref.save_trace_csv(str(tmp_path / "w.csv"), a, p, o, cls)
    for cls in (None, c[:0]):  # an empty trace: all_of(...) is true, the header has ",class"
        assert restate.trace_format(a[:0], p[:0], o[:0], cls) == \
            ref.save_trace_csv(str(tmp_path / "e.csv"), a[:0], p[:0], o[:0], cls)


def test_round_trip_generated_trace(restate):
    a, p, o = restate.gen_poisson_trace(5.0, 600_000, seed=4)
    cls = (p > 1024).astype(np.uint8)
    text = restate.trace_format(a, p, o, cls)
    r = restate.trace_parse(text, 1024)
    assert (r[0] == a).all() and (r[1] == p).all() and (r[2] == o).all() and (r[3] == cls).all()
    assert r[4] is True
