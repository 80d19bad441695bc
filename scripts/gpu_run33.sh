mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "index" > gpurun_out/pytest_capn.log 2>&1; echo t=$? > gpurun_out/status33.txt
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
for c in c3 c4; do WMH_INDEX_STATS=1 $B --config $c > gpurun_out/b33_$c.log 2>&1; done
echo done >> gpurun_out/status33.txt
