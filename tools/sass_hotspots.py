"""Per-source-line hot spots of one kernel from an ncu report + the local cubin's line info.
python tools/sass_hotspots.py REPORT.ncu-rep LIB.so KERNEL_SUBSTRING [top] [MANGLED_SUBSTRING]
(the first captured launch whose name matches KERNEL_SUBSTRING; MANGLED_SUBSTRING picks the
template instantiation in the cubin, e.g. k_route_binILi8ELi4ELb0E)
(ncu's own source view needs the build path; this maps SASS addresses with nvdisasm -g.)"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
mangled = sys.argv[5] if len(sys.argv) > 5 else kern
raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = raw.splitlines()
heads = [i for i, ln in enumerate(lines) if ln.startswith('"Kernel Name"')]
if len(heads) > 1:
    lines = lines[:heads[1]]
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ia, ie, ist = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
    "Warp Stall Sampling (All Samples)")
prof = {}
base = None
for r in rows[1:]:
    try:
        a = int(r[ia], 16)
    except (ValueError, IndexError):
        continue
    base = a if base is None else base  # ncu lists absolute addresses from the entry point
    prof[a - base] = (float(r[ie] or 0), float(r[ist] or 0))
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
addr2line = {}
for cub in os.listdir(d):
    sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True,
                          text=True).stdout
    cur, inside, loc = None, False, None
    for ln in sass.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln) or re.match(r"^(_Z\S+):$", ln)
        if m:
            inside = mangled in m.group(1)
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            loc = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and loc:
            addr2line[int(m.group(1), 16)] = loc
    if addr2line:
        break
agg = collections.defaultdict(lambda: [0.0, 0.0])
tot_i = sum(v[0] for v in prof.values())
tot_s = sum(v[1] for v in prof.values())
for a, (ni, ns) in prof.items():
    k = addr2line.get(a, ("?", 0))
    agg[k][0] += ni
    agg[k][1] += ns
print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
for k, (ni, ns) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:<5} inst {ni / tot_i * 100:6.2f}%  stall {ns / max(tot_s, 1) * 100:6.2f}%")
