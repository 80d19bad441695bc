mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bitplanes or (parity_configs and (tiled or auto))" > gpurun_out/pytest_b47.log 2>&1; echo t=$? > gpurun_out/status47.txt
B="timeout 1200 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --config c5 --gpu-gen"
WMH_TILED_STATS=1 $B > gpurun_out/b47_c5_auto.log 2>&1
WMH_TILED_BS=0 $B > gpurun_out/b47_c5_cm.log 2>&1
echo done >> gpurun_out/status47.txt
