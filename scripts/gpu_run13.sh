mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3"
for hc in 1 2 3 4 8; do WMH_CM_HCHUNKS=$hc $B > gpurun_out/b13_hc$hc.log 2>&1; done
echo done > gpurun_out/status13.txt
