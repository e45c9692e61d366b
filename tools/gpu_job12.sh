python tools/ab_variants.py 1024 single 65536 0,1,2,4 9
python tools/ab_variants.py 1024 single 131072 0,1,2,4 9
python tools/ab_variants.py 1024 single 524288 0,1 5
python tools/ab_variants.py 2048 single 65536 0,1,4 9
python tools/ab_variants.py 2048 double 32768 0,1,4 9
python tools/ab_variants.py 2048 double 131072 0,1,4 5
python tools/ab_variants.py 1024 double 65536 0,1,4 9
python tools/ab_variants.py 512 single 262144 0,1,2 9
