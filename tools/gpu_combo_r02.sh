# fp64 N=2048: combine the two data-pipe savers measured separately -- LDG + split re/im exchange
# (v12) and one-load twiddles (v13, TWP 3) -> v17 (and v18 with TWP 2) -- against the default (v0).
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -q -p no:cacheprovider -k "all_kernel_variants or every_real_capable or nonfinite_detection_every_variant" 2>&1 | tail -2
timeout 300 python tools/sweep.py --all-variants --cool 0.3 --n 2048 --prec double --json gpurun_out/r02_sweep_combo.json > /dev/null 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r02_sweep_combo.json'))
for p in (d if isinstance(d, list) else d.get('points', d)):
    if p['variant'] in (0, 12, 13, 17, 18): print(p['variant'], p['gbs'], p['frac'])
"
timeout 300 python tools/variant_accuracy.py 2>&1 | grep -E '"n": 2048' | grep -i double | grep -E '"variant": (0|12|13|17|18),'
timeout 600 python tools/sustained.py 2048 double 32768 copy,0,12,13,17,18 --secs 4 --rounds 3 2>&1 | tail -1
for v in 0 17 18; do NS=2048 VARIANT_DOUBLE_2048=$v timeout 120 python tools/real_input_probe.py 2>&1 | grep double; done
