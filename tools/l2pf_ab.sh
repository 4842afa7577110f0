# A/B of the L2 prefetch-size hints (wht_kernels.cuh: SV_L2_PF on the strided complex64 element loads,
# SV_L2_PF_V4 on the 128-bit loads); libs built with build.py -D... --out=abtmp/...
set -x
O=gpurun_out/l2pf2; mkdir -p $O
for rep in 1 2; do
for v in base pf0 v4; do
  if [ $v = base ]; then L=; else L=abtmp/libsv_$v.so; fi
  for cfg in c4 c3 c5w c3m; do
    SV_LIB=$L timeout 400 python bench.py --config $cfg --no-cpu-baseline > $O/bench_${cfg}_${v}_$rep.log 2>&1
  done
done
done
SV_LIB= timeout 600 python tools/gate_bench.py --out $O/gate_base.json > $O/gate_base.log 2>&1
SV_LIB=abtmp/libsv_pf0.so timeout 600 python tools/gate_bench.py --out $O/gate_pf0.json > $O/gate_pf0.log 2>&1
echo done
