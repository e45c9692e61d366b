# Is the sustained (power-capped) drop in the memory system or in the kernels? copy_ vs FFT under sustained load.
set -x
timeout 300 python tools/sustained.py 2048 double 32768 copy,0,4 --secs 5 --rounds 2 > gpurun_out/sus_copy_2048d.json 2>&1
timeout 300 python tools/sustained.py 1024 single 65536 copy,0 --secs 5 --rounds 2 > gpurun_out/sus_copy_1024s.json 2>&1
cat gpurun_out/sus_copy_*.json
