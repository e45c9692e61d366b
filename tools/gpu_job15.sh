nvidia-smi --query-gpu=index,clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks15.csv &
SMI=$!
python tools/ab_variants.py 1024 single 65536 0,1,3,6,7 7
python tools/ab_variants.py 2048 single 65536 0,3,5,6 7
kill $SMI
python tools/sweep.py --n 1024,2048 --prec single --all-variants > gpurun_out/sweep15.log 2>&1
