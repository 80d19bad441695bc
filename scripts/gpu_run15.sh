mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_real.py -m gpu -x -q > gpurun_out/pytest_real.log 2>&1; echo real=$? > gpurun_out/status15.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo all=$? >> gpurun_out/status15.txt
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b15_c2.log 2>&1; echo bench=$? >> gpurun_out/status15.txt
