# TMEM for the staging gather only (loader 4; variants 16 = no cap, 17 = 5 CTAs/SM) vs 0 and 14/15.
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "variant" 2>&1 | tail -1
python tools/sweep.py --prec double --n 2048 --all-variants --cool 0.3 2>&1 | grep -E '"variant": (0|14|15|16|17),'
python tools/sustained.py 2048 double 131072 copy,0,16,17 --secs 4 --rounds 3 2>&1 | tail -1
