set -x
mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "index" > gpurun_out/pytest_index.log 2>&1; echo pytest=$? > gpurun_out/status8.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 --algo index"
for cf in 0.25 0.5 1; do WMH_INDEX_CF=$cf $B > gpurun_out/b8_c2_cf$cf.log 2>&1; done
for cf in 0.25 0.5 1; do WMH_INDEX_CF=$cf $B --config c5 --rows 262144 --gpu-gen > gpurun_out/b8_c5_cf$cf.log 2>&1; done
for c in c3 c4; do $B --config $c --rows 65536 > gpurun_out/b8_${c}_64k.log 2>&1; done
CMD="python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 3 --algo index"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_index -s 3 -c 1 -o gpurun_out/prof8_index_c2 $CMD > gpurun_out/ncu8_c2.log 2>&1
echo done >> gpurun_out/status8.txt
