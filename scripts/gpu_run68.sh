mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "bitplanes" > gpurun_out/pytest_b68.log 2>&1; echo t=$? > gpurun_out/status68.txt
