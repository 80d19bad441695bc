mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bitplanes or (parity_configs and tiled)" > gpurun_out/pytest_b56.log 2>&1; echo t=$? > gpurun_out/status56.txt
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
$B --config c5 --rows 1000000 --gpu-gen > gpurun_out/b56_c5_1m.log 2>&1
WMH_TILED_BS=1 $B --config c2 > gpurun_out/b56_c2_bs.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --config c5 --gpu-gen > gpurun_out/b56_c5.log 2>&1
echo done >> gpurun_out/status56.txt
