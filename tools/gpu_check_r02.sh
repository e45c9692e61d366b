# Full GPU test suite + sanitizers over the TMA loaders + default sweep + bench, after kernel changes.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick --loader 1 2>&1 | tail -2
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_run.py --quick --loader 1 2>&1 | tail -2
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/r02_bench_check.json 2> gpurun_out/r02_bench_check.err
python tools/sustained.py 512 double 131072 copy,0,1 --secs 4 --rounds 3 2>&1
