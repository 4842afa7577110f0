# Regenerates the round's measured evidence on the GPU box (one B200):
#   gpurun -- 'bash tools/measure_round.sh'   then here:
#   python tools/ncu_summarize.py gpurun_out/r1b profiles r1
set -x
O=gpurun_out/r1b; mkdir -p $O
python bench.py > $O/bench_c4.log 2>&1
python bench.py --impl reference > $O/bench_ref_c4.log 2>&1
for cfg in c1 c2 c3 c3m c5w c5m c3n c4n c3d; do python bench.py --config $cfg --no-cpu-baseline > $O/bench_$cfg.log 2>&1; done
python tools/gate_bench.py --out $O/gate_bench.json > $O/gate_bench.log 2>&1
python tools/pass_breakdown.py --n 32 --k 4 > $O/pass_breakdown_n32.json 2>&1
python tools/pass_breakdown.py --n 28 --k 4 > $O/pass_breakdown_n28.json 2>&1
python tools/pass_breakdown.py --n 34 --k 2 > $O/pass_breakdown_n34.json 2>&1
python tools/whole_state_bench.py > $O/whole_state_bench.txt 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:wht_tile -s 65 -c 4 -o $O/c4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full.log 2>&1
