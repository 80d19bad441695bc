O=gpurun_out/r2_meas1
timeout 900 python bench.py > $O/bench_c5.json 2>$O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_c5_reference.json 2>$O/ref.err
timeout 300 python bench.py --config c1 --graph --steps 20 > $O/bench_c1_graph.json 2>/dev/null
timeout 300 python bench.py --config c2 > $O/bench_c2.json 2>/dev/null
timeout 900 python bench.py --config c3 --steps 5 > $O/bench_c3.json 2>/dev/null
timeout 900 python bench.py --config c4 --steps 5 > $O/bench_c4.json 2>/dev/null
for isg in table bsearch; do
 python scripts/kprobe.py --config c1 --rows 1000 --k 64 --algo simple --isgreen $isg >> $O/isgreen.txt 2>&1
 python scripts/kprobe.py --config c2 --rows 100000 --k 500 --algo simple --isgreen $isg >> $O/isgreen.txt 2>&1
 python scripts/kprobe.py --config c5 --rows 65536 --k 1024 --algo simple --isgreen $isg >> $O/isgreen.txt 2>&1
 python scripts/kprobe.py --config c5 --rows 1048576 --k 1024 --tile bitslice --isgreen $isg >> $O/isgreen.txt 2>&1
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --collide-pairs 0"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hash_bitslice -s 3 -c 1 -o $O/prof_c5 $CMD > $O/ncu_full.log 2>&1
echo done > $O/done.txt
