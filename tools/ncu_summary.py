"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py --rep gpurun_out/prof_c2.ncu-rep --workload "<config.workload>" \
        --out profiles/r01_ncu_c2.txt [--launches gpurun_out/launches_c2.csv]

Writes a human-readable metric dump and merges the per-launch DRAM traffic
into profiles/ncu_summary.json, keyed by bench.py's config.workload string
(bench.py reads `traffic` for the roofline object from there).
"""

import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__block_size",
    "launch__grid_size",
    "sm__cycles_elapsed.avg.per_second",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}  # -> us


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--workload", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--launches")
    args = ap.parse_args()
    lines = []
    summary = None
    for hdr, units, vals in raw(args.rep):
        rec = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        lines.append(f"kernel: {rec['Kernel Name'][0]}")
        for m in METRICS:
            if m in rec:
                lines.append(f"  {m} = {rec[m][0]} {rec[m][1]}")
        rd = float(rec["dram__bytes_read.sum"][0]) * SCALE.get(rec["dram__bytes_read.sum"][1], 1)
        wr = float(rec["dram__bytes_write.sum"][0]) * SCALE.get(rec["dram__bytes_write.sum"][1], 1)
        lines.append(f"  dram bytes read+write per launch = {rd + wr:.0f}")
        summary = {"kernel": rec["Kernel Name"][0], "dram_bytes_per_launch": rd + wr,
                   "dram_read": rd, "dram_write": wr, "source": os.path.basename(args.rep),
                   "duration_us_ncu": float(rec["gpu__time_duration.sum"][0]) * US.get(rec["gpu__time_duration.sum"][1], 1.0)}
    if args.launches:
        rows = [r for r in csv.DictReader(l for l in open(args.launches) if not l.startswith("=="))]
        agg = collections.defaultdict(list)
        for r in rows:
            agg[r["Kernel Name"]].append(float(r["Metric Value"]) * 1e3 * US.get(r.get("Metric Unit", "nsecond"), 1e-3))
        tot = sum(sum(v) for v in agg.values())
        lines.append("launch list (ncu gpu__time_duration.sum, cold-cache, serialised):")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"  {len(v):4d} x {sum(v) / len(v) / 1e3:9.2f} us  share {100 * sum(v) / tot:5.1f}%  {k[:110]}")
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    if summary:
        data[args.workload] = summary
    with open(path, "w") as f:
        json.dump(data, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
