mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
for nw in 1 2 4; do WMH_INDEX_NW=$nw WMH_INDEX_STATS=1 $B --config c3 > gpurun_out/b24_c3_nw$nw.log 2>&1; done
for nw in 1 2; do WMH_INDEX_NW=$nw WMH_INDEX_STATS=1 $B --algo index > gpurun_out/b24_c2_nw$nw.log 2>&1; done
for nw in 4 8; do WMH_INDEX_NW=$nw WMH_INDEX_STATS=1 $B --config c4 > gpurun_out/b24_c4_nw$nw.log 2>&1; done
WMH_INDEX_NW=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "index" > gpurun_out/pytest_nw1.log 2>&1; echo nw1=$? > gpurun_out/status24.txt
