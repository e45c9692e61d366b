nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks13.csv &
SMI=$!
python tools/ab_variants.py 1024 single 65536 0,1,4 9
python tools/ab_variants.py 2048 double 32768 0,1,4 9
python tools/ab_variants.py 1024 single 131072 0,1 7
kill $SMI
