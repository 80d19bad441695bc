set -x
mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "e2e" > gpurun_out/pytest_e2e.log 2>&1; echo pytest=$? > gpurun_out/status12.txt
timeout 900 python bench.py --config c5 --gpu-gen --steps 3 --warmup 3 --no-cpu-baseline --collide-pairs 10000000 > gpurun_out/b12_c5_auto.log 2>&1
timeout 900 python bench.py --config c5 --gpu-gen --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --algo index > gpurun_out/b12_c5_index.log 2>&1
for c in c3 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b12_${c}_e2e.log 2>&1; done
echo done >> gpurun_out/status12.txt
