# fp64 N=2048 with tensor-memory gathers (loader 3; variants 14 = no register cap, 15 = 5 CTAs/SM cap)
# against the default (0): parity + sanitizers, burst, sustained, real input, ncu.
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -p no:cacheprovider -k "variant or real" 2>&1 | tail -2
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_run.py --n 2048 --prec double 2>&1 | tail -2
done
python tools/sweep.py --prec double --n 2048 --all-variants --cool 0.3 2>&1 | grep -E '"variant": (0|13|14|15),'
python tools/sustained.py 2048 double 131072 copy,0,14,15 --secs 4 --rounds 3 2>&1 | tail -1
VARIANT_DOUBLE_2048=14 NS=2048 python tools/real_input_probe.py 2>&1 | grep double
VARIANT_DOUBLE_2048=15 NS=2048 python tools/real_input_probe.py 2>&1 | grep double
NS=2048 python tools/real_input_probe.py 2>&1 | grep double
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c4_tmem14 python tools/launch_variant.py 2048 double 131072 14 > gpurun_out/ncu_tmem14.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c4_tmem15 python tools/launch_variant.py 2048 double 131072 15 > gpurun_out/ncu_tmem15.log 2>&1
tail -1 gpurun_out/ncu_tmem14.log gpurun_out/ncu_tmem15.log
