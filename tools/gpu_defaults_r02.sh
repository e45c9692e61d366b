# After switching defaults (fp32 N=2048 -> R64 TMA, fp64 N=1024 -> R32 TMA): tests, sanitizers, sweeps, sustained.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick --loader 1 > gpurun_out/r02_sanitizer_racecheck_tma.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_run.py --quick --loader 1 > gpurun_out/r02_sanitizer_synccheck_tma.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py --quick > gpurun_out/r02_sanitizer_memcheck_defaults.txt 2>&1
tail -n 3 gpurun_out/r02_sanitizer_*.txt
NS=2,8,32,64,256,1024,2048 python tools/real_input_probe.py > gpurun_out/r02_real_input.jsonl 2>&1
for spec in "2048 single 65536 copy,0,1,8" "1024 double 65536 copy,0,1" "2048 double 32768 copy,0,7"; do
  python tools/sustained.py $spec --secs 4 --rounds 3 >> gpurun_out/r02_sustained_defaults.jsonl 2>&1
done
