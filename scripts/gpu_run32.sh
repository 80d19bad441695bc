mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
WMH_INDEX_NW=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m gpu -x -q -k "index or u16" > gpurun_out/pytest_indep.log 2>&1; echo t=$? > gpurun_out/status32.txt
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
for nw in 1 2; do WMH_INDEX_NW=$nw WMH_INDEX_STATS=1 $B --config c3 > gpurun_out/b32_c3_nw$nw.log 2>&1; done
for nw in 1 2; do WMH_INDEX_NW=$nw WMH_INDEX_STATS=1 $B --config c2r > gpurun_out/b32_c2r_nw$nw.log 2>&1; done
for nw in 1 2; do WMH_INDEX_NW=$nw WMH_INDEX_STATS=1 $B --algo index > gpurun_out/b32_c2_nw$nw.log 2>&1; done
echo done >> gpurun_out/status32.txt
