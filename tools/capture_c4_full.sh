# ncu --set full of 4 consecutive c4 tile passes (one iteration) at HEAD:  gpurun -- 'bash tools/capture_c4_full.sh'
set -x
O=gpurun_out/${MEAS_OUT:-r2i}; mkdir -p $O
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/plain_c4.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:wht_tile -s 65 -c 4 -o $O/c4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_c4_full.log 2>&1
echo "ncu rc=$?"; ls -la $O
