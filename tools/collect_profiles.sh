# Copy the round-end measurement set (tools/gpu_final_r02.sh output in gpurun_out/)
# into profiles/ under the round prefix, summarising the ncu captures, and
# print the DESIGN tables.   Usage: bash tools/collect_profiles.sh r02
set -e
cd "$(dirname "$0")/.."
R=${1:-r02}
W2="$(python -c "import bench; print(bench.CONFIGS['c2'][4])")"
W4="$(python -c "import bench; print(bench.CONFIGS['c4'][4])")"
W5="$(python -c "import bench; print(bench.CONFIGS['c5'][4])")"
python tools/ncu_summary.py --rep gpurun_out/prof_c2.ncu-rep --workload "$W2" --out profiles/${R}_ncu_c2.txt --launches gpurun_out/launches_c2.csv > /dev/null
python tools/ncu_summary.py --rep gpurun_out/prof_c4.ncu-rep --workload "$W4" --out profiles/${R}_ncu_c4.txt > /dev/null
python tools/ncu_summary.py --rep gpurun_out/prof_c5.ncu-rep --workload "$W5" --out profiles/${R}_ncu_c5.txt > /dev/null
python tools/ncu_summary.py --rep gpurun_out/prof_f2048.ncu-rep --workload "fp32 forward C2C FFT N=2048 batch=65536" --out profiles/${R}_ncu_f2048.txt > /dev/null
python tools/ncu_summary.py --rep gpurun_out/prof_d1024.ncu-rep --workload "fp64 forward C2C FFT N=1024 batch=65536" --out profiles/${R}_ncu_d1024.txt > /dev/null
for c in c2 c4 c5 f2048 d1024; do ncu -i gpurun_out/prof_$c.ncu-rep --page source --csv --print-source sass 2>/dev/null > gpurun_out/${c}_src.csv; done
(for c in c2 c4 c5 f2048 d1024; do echo "== $c"; python tools/ncu_stalls.py gpurun_out/${c}_src.csv 2>/dev/null | head -8; done) > profiles/${R}_ncu_stalls.txt
(for c in c4 f2048 d1024; do echo "== $c"; python tools/ncu_smem_excess.py gpurun_out/${c}_src.csv | tail -1; done) > profiles/${R}_ncu_smem.txt
for c in c2 c4 c5 c4_fill ref; do tail -n 1 gpurun_out/bench_$c.json > profiles/${R}_bench_$c.json; done
tail -n 1 gpurun_out/bench_c2_torchrun.json > profiles/${R}_bench_c2_torchrun_n1.json
cp gpurun_out/sweep_fwd.json profiles/${R}_sweep_fwd.json
cp gpurun_out/sweep_inv.json profiles/${R}_sweep_inv.json
cp gpurun_out/accuracy.json profiles/${R}_accuracy.json
cp gpurun_out/smoke.log profiles/${R}_smoke.log
cp gpurun_out/launches_c2.csv profiles/${R}_launches_c2.csv
cp gpurun_out/real_input.jsonl profiles/${R}_real_input.jsonl
cp gpurun_out/sustained_sweep.jsonl profiles/${R}_sustained_sweep.jsonl
tail -n 3 gpurun_out/pytest_gpu.log > profiles/${R}_pytest_gpu.txt
(for f in memcheck racecheck synccheck racecheck_tma racecheck_pipe; do echo "== sanitizer_$f.txt"; grep -v "^==PROF\|^$" gpurun_out/sanitizer_$f.txt | tail -n 3; done) > profiles/${R}_sanitizers.txt
python - "$R" <<'PY'
import json, sys
R = sys.argv[1]
for name in ("fwd", "inv"):
    rows = json.load(open(f"profiles/{R}_sweep_{name}.json"))
    for prec in ("single", "double"):
        rs = [r for r in rows if r["prec"] == prec]
        lab = "fp32" if prec == "single" else "fp64"
        print(f"{name} | {lab} GB/s | " + " | ".join(str(int(round(r["gbs"]))) for r in rs) + " |")
        print(f"{name} | {lab} ×copy | " + " | ".join("%.2f" % r["frac"] for r in rs) + " |")
        print(f"{name} | {lab} GFLOP/s | " + " | ".join(str(int(round(r["gflops"]))) for r in rs) + " |")
for c in ("c2", "c4", "c5", "c4_fill", "ref"):
    d = json.loads(open(f"profiles/{R}_bench_{c}.json").read())
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    print(c, d["value"], d["ms_per_step"], r.get("achieved"), r.get("frac"), r.get("kernel_ms"), e.get("value"),
          e.get("frac_of_link_bound"), (d.get("cpu_baseline") or {}).get("value"), (d.get("clocks") or {}).get("sm_mhz"),
          (d.get("clocks") or {}).get("reasons"))
for l in open(f"profiles/{R}_sustained_sweep.jsonl"):
    try:
        d = json.loads(l)
    except Exception:
        continue
    s = d["steady_gbs"]
    print("sustained", d["prec"], d["n"], s["-1"], s["0"], round(s["0"] / s["-1"], 3), d["sm_mhz"])
PY
