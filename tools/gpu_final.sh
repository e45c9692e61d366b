# Round-end measurement set: tests, smoke, bench lines, sweeps, accuracy, ncu, sanitizers, sustained.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,clocks_event_reasons.active --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config c5 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --no-cpu > gpurun_out/bench_c2_torchrun.json 2> gpurun_out/bench_c2_torchrun.err
timeout 600 python tools/sweep.py --cool 0.3 --json gpurun_out/sweep_fwd.json > gpurun_out/sweep_fwd.log 2>&1
timeout 600 python tools/sweep.py --cool 0.3 --dir inverse --json gpurun_out/sweep_inv.json > gpurun_out/sweep_inv.log 2>&1
timeout 600 python tests/accuracy_report.py gpurun_out/accuracy.json > gpurun_out/accuracy.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 1 --no-check > gpurun_out/ncu_launch_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 4 --warmup 3 --no-cpu --e2e-steps 1 --no-check > gpurun_out/ncu_full_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c4 python bench.py --config c4 --steps 4 --warmup 3 --no-cpu --e2e-steps 1 --no-check > gpurun_out/ncu_full_run_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c5 python bench.py --config c5 --steps 4 --warmup 3 --no-cpu --e2e-steps 1 --no-check > gpurun_out/ncu_full_run_c5.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/sanitizer_memcheck.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick > gpurun_out/sanitizer_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_run.py --quick > gpurun_out/sanitizer_synccheck.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick --loader 1 > gpurun_out/sanitizer_racecheck_tma.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick --loader 2 > gpurun_out/sanitizer_racecheck_pipe.txt 2>&1
timeout 300 python tools/sustained.py 1024 single 65536 copy,0 --secs 4 --rounds 2 > gpurun_out/sus_c2.json 2>&1
timeout 300 python tools/sustained.py 2048 double 131072 copy,0 --secs 4 --rounds 2 > gpurun_out/sus_c4.json 2>&1
timeout 300 python tools/sustained.py 512 single 262144 copy,0 --secs 4 --rounds 2 > gpurun_out/sus_c5.json 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
cat gpurun_out/smoke.log gpurun_out/bench_c2.json
