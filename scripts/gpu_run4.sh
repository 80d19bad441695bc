set -x
mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "index" > gpurun_out/pytest_index.log 2>&1; echo pytest=$? > gpurun_out/status4.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 --algo index"
WMH_INDEX_STATS=1 $B > gpurun_out/b4_c2.log 2>&1
for c in c3 c4; do WMH_INDEX_STATS=1 $B --config $c --rows 16384 > gpurun_out/b4_${c}.log 2>&1; done
WMH_INDEX_STATS=1 $B --config c5 --rows 262144 --gpu-gen > gpurun_out/b4_c5.log 2>&1
for c in c2 c3; do
CMD="python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 3 --config $c --rows 16384 --algo index"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${c}_index.csv $CMD > /dev/null 2>&1
done
CMD="python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 3 --algo index"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_index -s 3 -c 1 -o gpurun_out/prof_index_c2 $CMD > gpurun_out/ncu_c2.log 2>&1
echo done >> gpurun_out/status4.txt
