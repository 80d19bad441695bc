set -x
mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "index or auto" > gpurun_out/pytest_index.log 2>&1; echo pytest=$? > gpurun_out/status9.txt
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --algo index"
$B --config c5 --rows 262144 --gpu-gen > gpurun_out/b9_c5.log 2>&1
for c in c3 c4; do $B --config $c > gpurun_out/b9_${c}_full.log 2>&1; done
for c in c3 c4; do
CMD="python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 3 --config $c --rows 16384 --algo index"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches9_${c}_index.csv $CMD > /dev/null 2>&1
done
echo done >> gpurun_out/status9.txt
