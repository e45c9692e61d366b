# Default-variant selection under sustained load (and copy_ reference in the same run).
set -x
timeout 300 python tools/sustained.py 2048 single 65536 copy,0,5,4 --secs 4 --rounds 2 > gpurun_out/sel_2048s.json 2>&1
timeout 300 python tools/sustained.py 1024 double 65536 copy,0,1 --secs 4 --rounds 2 > gpurun_out/sel_1024d.json 2>&1
timeout 300 python tools/sustained.py 2048 double 32768 copy,0,4 --secs 4 --rounds 2 > gpurun_out/sel_2048d.json 2>&1
timeout 300 python tools/sustained.py 256 double 262144 copy,0,1 --secs 4 --rounds 2 > gpurun_out/sel_256d.json 2>&1
timeout 300 python tools/sustained.py 128 single 1048576 copy,0,1 --secs 4 --rounds 2 > gpurun_out/sel_128s.json 2>&1
timeout 300 python tools/sustained.py 32 single 4194304 copy,0 --secs 4 --rounds 2 > gpurun_out/sel_32s.json 2>&1
cat gpurun_out/sel_*.json
