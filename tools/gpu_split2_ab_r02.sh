# fp64 N=2048: R16 default (v0) vs split2 (v11) -- interleaved burst A/B, sustained, accuracy.
set -x
python tools/ab_variants.py 2048 double 32768 0,9,11 9
python tools/sustained.py 2048 double 32768 copy,0,11 --secs 4 --rounds 3
python tools/sustained.py 2048 double 131072 copy,0,11 --secs 4 --rounds 2
python tools/variant_accuracy.py 2>/dev/null | grep '"n": 2048' | grep double
