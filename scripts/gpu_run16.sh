mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo all=$? > gpurun_out/status16.txt
