mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m gpu -x -q -k "e2e or host" > gpurun_out/pytest_b43.log 2>&1; echo t=$? > gpurun_out/status43.txt
python scripts/e2e_probe.py > gpurun_out/e2e_ramp.json 2>&1
python scripts/e2e_probe.py > gpurun_out/e2e_ramp2.json 2>&1
WMH_E2E_CHUNKS=8 python scripts/e2e_probe.py > gpurun_out/e2e_u8.json 2>&1
echo done >> gpurun_out/status43.txt
