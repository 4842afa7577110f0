O=gpurun_out/r2l; mkdir -p $O
timeout 900 python tools/gate_bench.py --n 30 --reps 3 --out $O/gate_bench_final.json > $O/gb_final.log 2>&1; echo "gb rc=$?"
timeout 1500 python tools/costmodel_validate.py --out $O/costmodel_validation.json > $O/cm.log 2>&1; echo "cm rc=$?"
