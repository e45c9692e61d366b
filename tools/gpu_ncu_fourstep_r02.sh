set -x
for v in 16 9 0; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"fourstep|stockham" -s 2 -c 1 -o gpurun_out/prof_fs_v$v python tools/launch_variant.py 2048 double 32768 $v 3 > gpurun_out/ncu_fs_v$v.log 2>&1
done
ls -la gpurun_out
