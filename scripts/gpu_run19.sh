mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m gpu -x -q -k "tiled or auto or invariance" > gpurun_out/pytest_tiled.log 2>&1; echo pytest=$? > gpurun_out/status19.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3"
for r in 1 2; do WMH_CM_SWAR_ROUNDS=$r $B > gpurun_out/b19_c2_r$r.log 2>&1; done
for r in 1 2; do WMH_CM_SWAR_ROUNDS=$r $B --config c5 --rows 262144 --gpu-gen --algo tiled > gpurun_out/b19_c5_r$r.log 2>&1; done
echo done >> gpurun_out/status19.txt
