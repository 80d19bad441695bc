mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m gpu -x -q -k "index or auto or u16" > gpurun_out/pytest_index.log 2>&1; echo pytest=$? > gpurun_out/status25.txt
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
WMH_INDEX_STATS=1 $B --config c3 > gpurun_out/b25_c3.log 2>&1
WMH_INDEX_STATS=1 $B --config c4 > gpurun_out/b25_c4.log 2>&1
$B --algo index > gpurun_out/b25_c2.log 2>&1
echo done >> gpurun_out/status25.txt
