# HEAD verification on one B200 (short form of measure_final.sh):  gpurun -- 'bash tools/verify_head.sh'
set -x
O=gpurun_out/${MEAS_OUT:-r2h}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "gputest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py > $O/bench_c4.log 2>&1; echo "bench rc=$?"
timeout 300 python bench.py --impl reference > $O/bench_ref_c4.log 2>&1
for cfg in c1 c2 c3 c3m c5w c5m c3n c4n c3d; do timeout 400 python bench.py --config $cfg --no-cpu-baseline > $O/bench_$cfg.log 2>&1; done
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
tail -3 $O/gputest.log; tail -2 $O/smoke.log; tail -1 $O/bench_c4.log
echo done
