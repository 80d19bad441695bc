mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tiled or auto" > gpurun_out/pytest_t35.log 2>&1; echo t=$? > gpurun_out/status35.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 3"
$B > gpurun_out/b35_c2.log 2>&1
$B --config c5 --rows 262144 --gpu-gen > gpurun_out/b35_c5.log 2>&1
