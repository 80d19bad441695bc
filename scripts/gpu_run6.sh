set -x
mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "c3 or c4" > gpurun_out/pytest_full34.log 2>&1; echo pytest=$? > gpurun_out/status6.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --algo index"
for c in c3 c4; do for cf in 1 2 4 8 12 24; do WMH_INDEX_CF=$cf $B --config $c --rows 16384 > gpurun_out/b6_${c}_cf$cf.log 2>&1; done; done
for c in c3 c4; do for nw in 2 4 8; do WMH_INDEX_NW=$nw $B --config $c --rows 16384 > gpurun_out/b6_${c}_nw$nw.log 2>&1; done; done
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --config c4 > gpurun_out/b6_c4_full.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --config c3 > gpurun_out/b6_c3_full.log 2>&1
echo done >> gpurun_out/status6.txt
