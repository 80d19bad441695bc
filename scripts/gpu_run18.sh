mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_real.py -m gpu -q > gpurun_out/pytest_real.log 2>&1; echo real=$? > gpurun_out/status18.txt
timeout 600 python bench.py --config c2r > gpurun_out/b18_c2r.log 2>&1; echo c2r=$? >> gpurun_out/status18.txt
CMD="python bench.py --config c2r --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2r.csv $CMD > /dev/null 2>&1
