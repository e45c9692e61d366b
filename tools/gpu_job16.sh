nvidia-smi --query-gpu=index,clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks16.csv &
SMI=$!
python tools/ab_variants.py 1024 single 65536 0,1,4,7 11
python tools/ab_variants.py 1024 single 65536 7,4,1,0 11
kill $SMI
