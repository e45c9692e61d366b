# split2 with skewed staging (conflict-free polyphase gather): correctness, sanitizers, ncu smem, A/B.
set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_config_parity.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick --loader 1 2>&1 | tail -2
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_run.py --quick --loader 1 2>&1 | tail -2
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py --quick --loader 1 2>&1 | tail -2
B="python bench.py --steps 4 --warmup 3 --no-cpu --no-extras --e2e-steps 1 --no-check"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stockham|split2" -s 3 -c 1 -o gpurun_out/prof_c4 $B --config c4 > gpurun_out/ncu_c4.log 2>&1
python tools/sweep.py --all-variants --cool 0.3 --n 2048 --prec double --json gpurun_out/r02_sweep_split2.json > /dev/null 2>&1
NS=2048 python tools/real_input_probe.py 2>&1 | grep double
python tools/ab_variants.py 2048 double 32768 0,1,10 7
python tools/sustained.py 2048 double 32768 copy,0,1,10 --secs 4 --rounds 3
