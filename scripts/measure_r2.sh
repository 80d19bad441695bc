#!/bin/bash
# Round-2 end measurements (run through gpurun on one B200):
#   bash scripts/gpu_job.sh r2_end 'bash scripts/measure_r2.sh gpurun_out/r2_end'
O=${1:-gpurun_out/r2_end}
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -rs > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench_c5.json 2>$O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_c5_reference.json 2>$O/ref.err
timeout 300 python bench.py --config c1 --graph --steps 20 > $O/bench_c1_graph.json 2>/dev/null
timeout 300 python bench.py --config c2 > $O/bench_c2.json 2>/dev/null
timeout 600 python bench.py --config c2r > $O/bench_c2r.json 2>/dev/null
timeout 900 python bench.py --config c3 --steps 5 > $O/bench_c3.json 2>/dev/null
timeout 900 python bench.py --config c4 --steps 5 > $O/bench_c4.json 2>/dev/null
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --collide-pairs 0"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hash_bitslice -s 3 -c 1 -o $O/prof_c5 $CMD > $O/ncu_c5.log 2>&1
CMD3="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:hash_index -s 3 -c 1 -o $O/prof_c3 $CMD3 > $O/ncu_c3.log 2>&1
CMD2="python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:hash_tiled_cm -s 3 -c 1 -o $O/prof_c2 $CMD2 > $O/ncu_c2.log 2>&1
echo done > $O/done.txt
