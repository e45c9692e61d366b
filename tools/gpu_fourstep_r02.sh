# fp64 N=2048 four-step kernel (32 x 64, one exchange, three shuffle radix-2 levels, 128 threads):
# variants 16 (5 CTAs/SM) and 17 (4 CTAs/SM) against the R16 default (0) and R32 two-warp (9).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -q -p no:cacheprovider -k "all_kernel_variants or every_real_capable or nonfinite_detection_every_variant" 2>&1 | tail -4
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick --n 2048 --prec double 2>&1 | tail -2
timeout 300 python tools/sweep.py --all-variants --cool 0.3 --n 2048 --prec double --json gpurun_out/r02_sweep_fourstep.json > /dev/null 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r02_sweep_fourstep.json'))
for p in (d if isinstance(d, list) else d.get('points', d)):
    if p['variant'] in (0, 9, 11, 16, 17): print(p)
" 2>&1 | head -40
for v in 0 16 17; do NS=2048 VARIANT_DOUBLE_2048=$v timeout 120 python tools/real_input_probe.py 2>&1 | grep double; done
timeout 300 python tools/variant_accuracy.py 2>&1 | grep -E '"n": 2048' | grep -i double | grep -E '"variant": (0|16|17),'
timeout 400 python tools/sustained.py 2048 double 32768 copy,0,9,16,17 --secs 4 --rounds 3 > gpurun_out/r02_sustained_fourstep.jsonl 2>&1
tail -3 gpurun_out/r02_sustained_fourstep.jsonl
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"fourstep" -s 2 -c 1 -o gpurun_out/prof_fs4_v16 python tools/launch_variant.py 2048 double 32768 16 3 > gpurun_out/ncu_fs4.log 2>&1
