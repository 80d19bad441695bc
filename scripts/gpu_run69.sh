mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "bitplanes" > gpurun_out/pytest_b69.log 2>&1; echo t=$? > gpurun_out/status69.txt
timeout 1200 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --config c5 --gpu-gen > gpurun_out/b69_c5.log 2>&1
echo done >> gpurun_out/status69.txt
