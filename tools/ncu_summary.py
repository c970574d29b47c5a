"""Summarise ncu reports / launch lists into profiles/ (markdown + JSON).

  python tools/ncu_summary.py report <file.ncu-rep> <out_prefix>
  python tools/ncu_summary.py launches <launches.csv> <out.md>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
    "lts__t_bytes.sum": "l2_bytes",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for m, k in METRICS.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                u = units[hdr.index(m)]
                try:
                    val = float(v)
                except ValueError:
                    continue
                if u == "Kbyte":
                    val *= 1e3
                elif u == "Mbyte":
                    val *= 1e6
                elif u == "Gbyte":
                    val *= 1e9
                elif u in ("usecond", "us"):
                    val *= 1e3
                elif u in ("msecond", "ms"):
                    val *= 1e6
                d[k] = val
        stalls = []
        for h, v in zip(hdr, r):
            if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(v), h.split("stalled_")[1].split("_per_issue")[0]))
                except ValueError:
                    pass
        d["top_stalls"] = [f"{n}={x:.2f}" for x, n in sorted(stalls, reverse=True)[:5]]
        res.append(d)
    return res


def report(rep, prefix):
    res = raw(rep)
    with open(prefix + ".json", "w") as f:
        json.dump(res, f, indent=1)
    lines = [f"# ncu --set full summary: `{rep.split('/')[-1]}`", "",
             "| kernel | dur (us) | DRAM R+W (MB) | DRAM % | SM % | FP64 pipe % | occ % | regs | top stalls |",
             "|---|---|---|---|---|---|---|---|---|"]
    for d in res:
        rw = (d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)) / 1e6
        lines.append(f"| {d['kernel'][:60]} | {d.get('duration_ns', 0) / 1e3:.1f} | {rw:.2f} | "
                     f"{d.get('dram_pct', 0):.1f} | {d.get('sm_pct', 0):.1f} | {d.get('fp64_pipe_pct', 0):.1f} | "
                     f"{d.get('achieved_occupancy_pct', 0):.1f} | {d.get('registers', 0):.0f} | "
                     f"{', '.join(d['top_stalls'])} |")
    open(prefix + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi, ni = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        if r[ni] == "gpu__time_duration.sum":
            agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# launch list `{path.split('/')[-1]}` (ncu gpu__time_duration, cold-cache, serialised)", "",
             "| kernel | launches | mean (us) | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / tot * 100:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:20]))


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2], sys.argv[3])
    else:
        launches(sys.argv[2], sys.argv[3])
