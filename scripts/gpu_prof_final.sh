mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
for c in c3 c4; do
CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_final_$c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_index -s 3 -c 1 -o gpurun_out/prof_final_$c $CMD > gpurun_out/ncu_final_$c.log 2>&1
CMD2="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD2 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final_$c.csv $CMD2 > /dev/null 2>&1
done
echo done > gpurun_out/status_pf.txt
