O=gpurun_out/final8
mkdir -p $O
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python bench.py --config c4 --steps 5 > $O/bench_c4.json 2>/dev/null
timeout 900 python bench.py --config c3 --steps 5 > $O/bench_c3.json 2>/dev/null
timeout 600 python bench.py --config c2r > $O/bench_c2r.json 2>/dev/null
CMD2="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD2 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv $CMD2 > /dev/null 2>&1
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_index -s 3 -c 1 -o $O/prof_c4 $CMD > $O/ncu_c4.log 2>&1
echo done > $O/status.txt
