# Round-2 final measured evidence on one B200:  gpurun -- 'bash tools/measure_final.sh'
set -x
O=gpurun_out/r2f; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "gputest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py > $O/bench_c4.log 2>&1
timeout 300 python bench.py --impl reference > $O/bench_ref_c4.log 2>&1
for cfg in c1 c2 c3 c3m c5w c5m c3n c4n c3d; do timeout 400 python bench.py --config $cfg --no-cpu-baseline > $O/bench_$cfg.log 2>&1; done
timeout 300 python tools/sample_bench.py --n 32 --reps 3 > $O/sample_n32.json 2>&1
timeout 300 python tools/whole_state_bench.py > $O/whole_state.txt 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 300 python bench.py --config c5m --steps 1 --warmup 1 --no-cpu-baseline > $O/plain_c5m.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:mean_tile -s 2 -c 1 -o $O/c5m_mean_full python bench.py --config c5m --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_c5m.log 2>&1
echo done
