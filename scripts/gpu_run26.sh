mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
for nw in 2 4; do WMH_INDEX_NW=$nw WMH_INDEX_STATS=1 $B --config c3 > gpurun_out/b26_c3_nw$nw.log 2>&1; done
WMH_INDEX_STATS=1 $B --config c4 > gpurun_out/b26_c4.log 2>&1
