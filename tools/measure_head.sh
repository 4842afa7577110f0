# Re-verify HEAD on one B200 after a container re-creation:  gpurun -- 'bash tools/measure_head.sh'
set -x
O=gpurun_out/r2h; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "gputest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py > $O/bench_c4.log 2>&1
for cfg in c2 c5w; do timeout 400 python bench.py --config $cfg --no-cpu-baseline > $O/bench_$cfg.log 2>&1; done
echo done
