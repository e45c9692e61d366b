# Round-2 measurement set: tests, smoke, bench lines, sweeps, accuracy, ncu, sanitizers, sustained.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,clocks_event_reasons.active --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu --no-extras > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config c5 --no-cpu --no-extras > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --config c4 --fill-hbm 0.9 --steps 10 --warmup 3 --no-cpu --no-extras --e2e-steps 1 > gpurun_out/bench_c4_fill.json 2> gpurun_out/bench_c4_fill.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --no-cpu --no-extras > gpurun_out/bench_c2_torchrun.json 2> gpurun_out/bench_c2_torchrun.err
timeout 600 python tools/sweep.py --cool 0.3 --json gpurun_out/sweep_fwd.json > gpurun_out/sweep_fwd.log 2>&1
timeout 600 python tools/sweep.py --cool 0.3 --dir inverse --json gpurun_out/sweep_inv.json > gpurun_out/sweep_inv.log 2>&1
timeout 600 python tests/accuracy_report.py gpurun_out/accuracy.json > gpurun_out/accuracy.log 2>&1
NS=2,8,32,64,256,512,1024,2048 timeout 600 python tools/real_input_probe.py > gpurun_out/real_input.jsonl 2>&1
B="python bench.py --steps 4 --warmup 3 --no-cpu --no-extras --e2e-steps 1 --no-check"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 10 --warmup 3 --no-cpu --no-extras --e2e-steps 1 --no-check > gpurun_out/ncu_launch_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stockham|split2" -s 3 -c 1 -o gpurun_out/prof_c2 $B > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stockham|split2" -s 3 -c 1 -o gpurun_out/prof_c4 $B --config c4 > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stockham|split2" -s 3 -c 1 -o gpurun_out/prof_c5 $B --config c5 > gpurun_out/ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stockham|split2" -s 3 -c 1 -o gpurun_out/prof_f2048 $B --n 2048 --precision single > gpurun_out/ncu_f2048.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stockham|split2" -s 3 -c 1 -o gpurun_out/prof_d1024 $B --n 1024 --precision double > gpurun_out/ncu_d1024.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/sanitizer_memcheck.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick > gpurun_out/sanitizer_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_run.py --quick > gpurun_out/sanitizer_synccheck.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick --loader 1 > gpurun_out/sanitizer_racecheck_tma.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick --loader 2 > gpurun_out/sanitizer_racecheck_pipe.txt 2>&1
timeout 1200 bash tools/sustained_sweep.sh > gpurun_out/sustained_sweep.jsonl 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
cat gpurun_out/smoke.log gpurun_out/bench_c2.json | cut -c1-400
