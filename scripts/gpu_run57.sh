mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 --config c2"
$B > gpurun_out/b57_base.log 2>&1
WMH_CM_HCHUNKS=1 $B > gpurun_out/b57_h1.log 2>&1
WMH_CM_HCHUNKS=4 $B > gpurun_out/b57_h4.log 2>&1
$B --chunk 16 > gpurun_out/b57_c16.log 2>&1
WMH_TILED_BS=1 WMH_BS_GROUPS=8 $B > gpurun_out/b57_bs8.log 2>&1
echo done > gpurun_out/status57.txt
