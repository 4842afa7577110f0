# Round-2 final measured evidence on one B200:  gpurun -- 'bash tools/measure_final.sh'
set -x
O=gpurun_out/${MEAS_OUT:-r2g}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "gputest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py > $O/bench_c4.log 2>&1
timeout 300 python bench.py --impl reference > $O/bench_ref_c4.log 2>&1
for cfg in c1 c2 c3 c3m c5w c5m c3n c4n c3d; do timeout 400 python bench.py --config $cfg --no-cpu-baseline > $O/bench_$cfg.log 2>&1; done
timeout 300 python tools/mean_resident_scan.py > $O/mean_resident_scan.jsonl 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 300 python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline > $O/plain_c2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:mean_resreg -s 1 -c 1 -o $O/c2_resreg_full python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 600 python tools/gate_bench.py --out $O/gate_bench_n30.json > $O/gate_bench.log 2>&1
timeout 300 python tools/pass_breakdown.py --n 32 --k 4 > $O/pass_breakdown_n32.json 2> $O/pass_breakdown.err
echo done
