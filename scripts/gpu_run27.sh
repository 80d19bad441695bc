mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3"
$B > gpurun_out/b27_c2.log 2>&1
$B --config c5 --rows 262144 --gpu-gen > gpurun_out/b27_c5.log 2>&1
