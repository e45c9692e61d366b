# Power-capped steady state for every N x precision (default kernel vs copy_), 1 GiB in.
for prec in single double; do
  esz=8; [ "$prec" = double ] && esz=16
  for p in 1 2 3 4 5 6 7 8 9 10 11; do
    n=$((1 << p)); rows=$(( (1 << 30) / (n * esz) ))
    timeout 120 python tools/sustained.py $n $prec $rows copy,0 --secs 3 --rounds 1
  done
done
