mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m gpu -x -q -k "tiled or auto or invariance" > gpurun_out/pytest_tiled.log 2>&1; echo pytest=$? > gpurun_out/status20.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3"
for tw in 1 2; do WMH_CM_TW=$tw $B > gpurun_out/b20_c2_tw$tw.log 2>&1; done
for tw in 1 2; do WMH_CM_TW=$tw $B --config c5 --rows 262144 --gpu-gen --algo tiled > gpurun_out/b20_c5_tw$tw.log 2>&1; done
for tw in 1 2; do WMH_CM_TW=$tw WMH_CM_SWAR_ROUNDS=2 $B > gpurun_out/b20_c2_tw${tw}_r2.log 2>&1; done
echo done >> gpurun_out/status20.txt
