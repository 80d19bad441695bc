O=gpurun_out/final7
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$? > $O/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/status.txt
timeout 600 python bench.py > $O/bench_c2.json 2>$O/bench_c2.err; echo bench=$? >> $O/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_c2_reference.json 2>/dev/null
timeout 300 python bench.py --config c1 > $O/bench_c1.json 2>/dev/null
timeout 600 python bench.py --config c2r > $O/bench_c2r.json 2>/dev/null
timeout 900 python bench.py --config c3 --steps 5 > $O/bench_c3.json 2>/dev/null
timeout 900 python bench.py --config c4 --steps 5 > $O/bench_c4.json 2>/dev/null
timeout 1200 python bench.py --config c5 --gpu-gen --steps 3 --collide-pairs 10000000 > $O/bench_c5.json 2>/dev/null
echo benches=done >> $O/status.txt
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv $CMD > /dev/null 2>&1
for c in c3 c4; do
CMD2="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD2 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv $CMD2 > /dev/null 2>&1
done
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:x3_ -s 4 -c 4 -o $O/prof_c4_build $CMD > $O/ncu_c4_build.log 2>&1
echo done >> $O/status.txt
CMD="python bench.py --config c5 --gpu-gen --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_tiled -s 3 -c 1 -o $O/prof_c5 $CMD > $O/ncu_c5.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_tiled -s 3 -c 1 -o $O/prof_c2 $CMD > $O/ncu_c2.log 2>&1
echo done2 >> $O/status.txt
for c in c3 c4; do
CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_index -s 3 -c 1 -o $O/prof_$c $CMD > $O/ncu_$c.log 2>&1
done
echo done3 >> $O/status.txt
