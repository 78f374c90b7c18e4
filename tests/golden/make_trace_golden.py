"""Writes tests/golden/trace_cases.json: greensim::load_trace's own result on every fixture of
tests/trace_cases.py (the reference library, oracle/_ref, needs /root/reference to build).
Run: python tests/golden/make_trace_golden.py"""
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.oracle import Reference  # noqa: E402
from trace_cases import CASES  # noqa: E402


def main():
    ref = Reference()
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, data, thr in CASES:
            f = os.path.join(d, "t.csv")
            with open(f, "wb") as fh:
                fh.write(data)
            r = ref.load_trace(f, thr)
            if isinstance(r[0], str):
                out[name] = {"error": [r[1], r[2], r[3]]}
            else:
                out[name] = {"arrival": [int(x) for x in r[0]], "prompt": [int(x) for x in r[1]],
                             "output": [int(x) for x in r[2]], "cls": [int(x) for x in r[3]]}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "trace_cases.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
