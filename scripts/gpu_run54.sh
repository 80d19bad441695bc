mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m gpu -x -q -k "index or auto or u16 or e2e or hasher or sharding" > gpurun_out/pytest_b54.log 2>&1; echo t=$? > gpurun_out/status54.txt
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
$B --config c4 > gpurun_out/b54_c4.log 2>&1
$B --config c3 > gpurun_out/b54_c3.log 2>&1
CMD="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b54_c4.csv $CMD > /dev/null 2>&1
echo done >> gpurun_out/status54.txt
