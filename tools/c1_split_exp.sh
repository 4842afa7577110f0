set -x
O=gpurun_out/c1exp; mkdir -p $O
for w in 3 4 5; do SV_WHOLE_W=$w timeout 300 python tools/whole_state_bench.py > $O/wsb_w$w.txt 2>&1; done
timeout 900 python -m pytest tests/test_whole_reg_gpu.py -q -p no:cacheprovider > $O/test.log 2>&1; echo "test rc=$?"
