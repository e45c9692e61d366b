# Copy the round-end measurement set (tools/gpu_final.sh output in gpurun_out/)
# into profiles/ under the round prefix, summarising the ncu captures, and
# print the DESIGN tables.   Usage: bash tools/collect_profiles.sh r01
set -e
cd "$(dirname "$0")/.."
R=${1:-r01}
W2="$(python -c "import bench; print(bench.CONFIGS['c2'][4])")"
W4="$(python -c "import bench; print(bench.CONFIGS['c4'][4])")"
W5="$(python -c "import bench; print(bench.CONFIGS['c5'][4])")"
python tools/ncu_summary.py --rep gpurun_out/prof_c2.ncu-rep --workload "$W2" --out profiles/${R}_ncu_c2.txt --launches gpurun_out/launches_c2.csv > /dev/null
python tools/ncu_summary.py --rep gpurun_out/prof_c4.ncu-rep --workload "$W4" --out profiles/${R}_ncu_c4.txt > /dev/null
python tools/ncu_summary.py --rep gpurun_out/prof_c5.ncu-rep --workload "$W5" --out profiles/${R}_ncu_c5.txt > /dev/null
for c in c2 c4 c5; do ncu -i gpurun_out/prof_$c.ncu-rep --page source --csv --print-source sass 2>/dev/null > gpurun_out/${c}_src.csv; done
(for c in c2 c4 c5; do echo "== $c"; python tools/ncu_stalls.py gpurun_out/${c}_src.csv 2>/dev/null | head -8; done) > profiles/${R}_ncu_stalls.txt
for c in c2 c4 c5 ref; do tail -n 1 gpurun_out/bench_$c.json > profiles/${R}_bench_$c.json; done
tail -n 1 gpurun_out/bench_c2_torchrun.json > profiles/${R}_bench_c2_torchrun_n1.json
cp gpurun_out/sweep_fwd.json profiles/${R}_sweep_fwd.json
cp gpurun_out/sweep_inv.json profiles/${R}_sweep_inv.json
cp gpurun_out/accuracy.json profiles/${R}_accuracy.json
cp gpurun_out/smoke.log profiles/${R}_smoke.log
cp gpurun_out/launches_c2.csv profiles/${R}_launches_c2.csv
(for f in memcheck racecheck synccheck racecheck_tma racecheck_pipe; do echo "== sanitizer_$f.txt"; grep -v "^==PROF\|^$" gpurun_out/sanitizer_$f.txt | tail -n 3; done) > profiles/${R}_sanitizers.txt
cat gpurun_out/sus_c2.json gpurun_out/sus_c4.json gpurun_out/sus_c5.json > profiles/${R}_sustained_defaults.jsonl
python - "$R" <<'PY'
import json, sys
R = sys.argv[1]
for name in ("fwd", "inv"):
    rows = json.load(open(f"profiles/{R}_sweep_{name}.json"))
    for prec in ("single", "double"):
        rs = [r for r in rows if r["prec"] == prec]
        lab = "fp32" if prec == "single" else "fp64"
        print(f"{name} | {lab} GB/s | " + " | ".join(str(int(round(r["gbs"]))) for r in rs) + " |")
        print(f"{name} | {lab} ×8 TB/s | " + " | ".join("%.2f" % (r["gbs"] / 8000) for r in rs) + " |")
        print(f"{name} | {lab} GFLOP/s | " + " | ".join(str(int(round(r["gflops"]))) for r in rs) + " |")
        print(f"{name} {lab} x copy range", min(r["frac"] for r in rs), max(r["frac"] for r in rs))
for c in ("c2", "c4", "c5", "ref"):
    d = json.loads(open(f"profiles/{R}_bench_{c}.json").read())
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    print(c, d["value"], d["ms_per_step"], r.get("achieved"), r.get("frac"), r.get("kernel_ms"), e.get("value"),
          e.get("frac_of_link_bound"), (d.get("cpu_baseline") or {}).get("value"))
PY
