mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
$B --config c5 --rows 1000000 --gpu-gen --algo tiled > gpurun_out/b37_c5_tiled.log 2>&1
$B --config c5 --rows 1000000 --gpu-gen --algo index > gpurun_out/b37_c5_index.log 2>&1
for h in 64 128 256 512; do $B --config c5 --rows 1000000 --gpu-gen --algo index --horizon $h > gpurun_out/b37_c5_index_h$h.log 2>&1; done
$B --config c2 --algo index > gpurun_out/b37_c2_index.log 2>&1
$B --config c2 --algo tiled > gpurun_out/b37_c2_tiled.log 2>&1
CMD="python bench.py --config c5 --rows 262144 --gpu-gen --algo index --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b37_c5.csv $CMD > /dev/null 2>&1
echo done > gpurun_out/status37.txt
