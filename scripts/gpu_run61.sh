mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m gpu -q -x -k "key_space or maximum or index or auto or e2e or hasher" > gpurun_out/pytest_b61.log 2>&1; echo t=$? > gpurun_out/status61.txt
