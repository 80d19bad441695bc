mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bitplanes or (parity_configs and (tiled or auto)) or edge or seeds or saturation" > gpurun_out/pytest_b38.log 2>&1; echo t=$? > gpurun_out/status38.txt
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
WMH_TILED_STATS=1 $B --config c2 --algo tiled > gpurun_out/b38_c2_bs.log 2>&1
WMH_TILED_BS=0 $B --config c2 --algo tiled > gpurun_out/b38_c2_cm.log 2>&1
WMH_TILED_STATS=1 $B --config c5 --rows 1000000 --gpu-gen --algo tiled > gpurun_out/b38_c5_bs.log 2>&1
WMH_TILED_BS=0 $B --config c5 --rows 1000000 --gpu-gen --algo tiled > gpurun_out/b38_c5_cm.log 2>&1
echo done >> gpurun_out/status38.txt
