mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 --config c2"
$B > gpurun_out/b58_base.log 2>&1
WMH_CM_TW=2 $B > gpurun_out/b58_tw2.log 2>&1
echo done > gpurun_out/status58.txt
