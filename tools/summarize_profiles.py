"""Turn gpurun_out/<round>_* ncu outputs into the committed evidence under profiles/:
  profiles/<round>_launches.csv     raw launch list (gpu__time_duration per launch)
  profiles/<round>_launch_summary.md per-kernel mean device time and share of the bench run
  profiles/<round>_kernels.md        key `--set full` metrics per captured kernel
  profiles/<round>_traffic.json      dram bytes / launch and duration of each captured kernel
usage: python tools/summarize_profiles.py r1
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_pct_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "warp_insts",
    "smsp__inst_executed_pipe_fp64.sum": "fp64_insts",
    "sm__cycles_active.avg": "sm_cycles_active",
}
UNIT_SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
              "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6,
              "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launch_summary(rnd):
    src = os.path.join(OUT, f"{rnd}_launches.csv")
    shutil.copy(src, os.path.join(PROF, f"{rnd}_launches.csv"))
    rows = list(csv.reader(open(src)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")].append(
                float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1e-3))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# {rnd} launch list summary (ncu gpu__time_duration.sum, --clock-control none;",
             "# cold-cache and serialised: compare shares, not absolute times)", "",
             "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.2f} | {sum(v):.1f} | {sum(v)/tot:.1%} |")
    open(os.path.join(PROF, f"{rnd}_launch_summary.md"), "w").write("\n".join(lines) + "\n")


def rep_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "").split("(")[0].replace("void ", "")
               .replace("<unnamed>::", "")}
        for m, k in METRICS.items():
            if m in d and d[m] not in ("", "n/a"):
                u = units[hdr.index(m)]
                try:
                    rec[k] = float(d[m].replace(",", "")) * UNIT_SCALE.get(u, 1.0)
                except ValueError:
                    pass
        out.append(rec)
    return out


def fp64_insts(rep, kernel):
    """FP64-pipe warp instructions (DFMA/DMUL/DADD/DSETP executed) of the first captured launch
    of `kernel`, summed from the report's per-SASS-instruction counts."""
    raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kernel, "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    lines = raw.splitlines()
    heads = [i for i, ln in enumerate(lines) if ln.startswith('"Kernel Name"')]
    if not heads:
        return None
    body = lines[heads[0] + 1:heads[1] if len(heads) > 1 else len(lines)]
    rows = list(csv.reader(io.StringIO("\n".join(body))))
    hdr = rows[0]
    isrc, ie = hdr.index("Source"), hdr.index("Instructions Executed")
    n = 0.0
    for r in rows[1:]:
        if len(r) <= ie:
            continue
        op = r[isrc].split()
        op = (op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else ""))
        if op.split(".")[0] in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"):
            n += float(r[ie] or 0)
    return n


def main(rnd):
    os.makedirs(PROF, exist_ok=True)
    launch_summary(rnd)
    recs = []
    for part in ("prefill", "decode", "pool"):
        rep = os.path.join(OUT, f"{rnd}_{part}.ncu-rep")
        if os.path.exists(rep):
            recs += [dict(r, part=part) for r in rep_metrics(rep)]
    lines = [f"# {rnd} ncu --set full captures (key metrics per launch)", "",
             "| kernel | us | DRAM R+W MB | DRAM % | SM % | FP64 pipe % (active) | issue % (active) | occupancy % | regs | warp insts |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    units_path = os.path.join(OUT, f"{rnd}_units.json")
    units = json.load(open(units_path)) if os.path.exists(units_path) else {}
    for r in recs:
        mb = (r.get("dram_read", 0) + r.get("dram_write", 0)) / 1e6
        lines.append(f"| `{r['kernel']}` | {r.get('duration', 0):.1f} | {mb:.2f} | "
                     f"{r.get('dram_pct', 0):.1f} | {r.get('sm_pct', 0):.1f} | "
                     f"{r.get('fp64_pipe_pct_active', 0):.1f} | {r.get('issue_pct_active', 0):.1f} | "
                     f"{r.get('occupancy_pct', 0):.1f} | {r.get('regs', 0):.0f} | "
                     f"{r.get('warp_insts', 0):.3g} |")
        rec = {"dram_bytes_per_launch": mb * 1e6, "duration_us": r.get("duration", 0),
               "warp_insts": r.get("warp_insts"), "fp64_insts": r.get("fp64_insts"),
               "fp64_pipe_pct_active": r.get("fp64_pipe_pct_active"),
               "issue_pct_active": r.get("issue_pct_active")}
        u = next((v for k, v in units.items() if r["kernel"].startswith(k)), None)
        if u:
            rec["units"] = u
        if r["part"] == "pool" and r["kernel"] in traffic:
            # K5's full-ring replay launch belongs to the same scenarios: add it in
            t = traffic[r["kernel"]]
            for k in ("dram_bytes_per_launch", "duration_us", "warp_insts"):
                t[k] = (t.get(k) or 0) + (rec.get(k) or 0)
            t["launches"] = t.get("launches", 1) + 1
        traffic.setdefault(r["kernel"], rec)
    open(os.path.join(PROF, f"{rnd}_kernels.md"), "w").write("\n".join(lines) + "\n")
    prep = os.path.join(OUT, f"{rnd}_prefill.ncu-rep")
    for k in list(traffic):
        if k.startswith("k_prefill_select") or k.startswith("k_route_bin"):
            base = k.split("<")[0]
            traffic[k]["fp64_insts"] = fp64_insts(prep, base) if os.path.exists(prep) else None
    json.dump(traffic, open(os.path.join(PROF, f"{rnd}_traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
