# Round-2 second batch on one B200:  gpurun -- 'bash tools/measure_round2b.sh'
set -x
O=gpurun_out/r2b; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "gputest rc=$?"
timeout 600 python tools/gate_bench.py --out $O/gate_bench_n30.json > $O/gate_bench.log 2>&1
SV_GATE_JIT=0 timeout 600 python tools/gate_bench.py --out $O/gate_bench_n30_interp.json > $O/gate_bench_interp.log 2>&1
timeout 1200 python tools/costmodel_validate.py --out $O/costmodel_validation.json > $O/costmodel.log 2>&1; echo "costmodel rc=$?"
SV_GATE_JIT=1 timeout 300 python tools/gate_profile_run.py qft > $O/gp_plain.log 2>&1 && SV_GATE_JIT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sv_gate_jit -s 5 -c 2 -o $O/gate_jit_qft python tools/gate_profile_run.py qft > $O/ncu_gate_jit.log 2>&1
SV_GATE_JIT=1 timeout 300 python tools/gate_profile_run.py u_layer > $O/gp_plain2.log 2>&1 && SV_GATE_JIT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sv_gate_jit -s 3 -c 1 -o $O/gate_jit_ulayer python tools/gate_profile_run.py u_layer > $O/ncu_gate_jit2.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/plain_c4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:wht_tile -s 65 -c 4 -o $O/c4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_c4_full.log 2>&1
timeout 300 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > $O/plain_c3.log 2>&1 && timeout 600 ncu --nvtx --nvtx-include "sv.wht_tile/" --metrics gpu__time_duration.sum -c 6 --csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_nvtx_c3.log 2>&1
echo done
