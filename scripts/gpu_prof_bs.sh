mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_tiled_bs -s 3 -c 1 -o gpurun_out/prof_c2_bs1 $CMD > gpurun_out/ncu_c2_bs1.log 2>&1
echo done > gpurun_out/status_pbs.txt
