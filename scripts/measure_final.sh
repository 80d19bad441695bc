#!/bin/bash
# Final refresh of the round-2 measurements on HEAD (trimmed measure_r2.sh; the
# c5 and c2 ncu captures in profiles/r2_end stay valid, their kernels are unchanged):
#   gpurun --timeout 2700 -- bash scripts/gpu_job.sh r2_final 'bash scripts/measure_final.sh gpurun_out/r2_final'
O=${1:-gpurun_out/r2_final}
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_c5.json 2>$O/bench_c5.err
timeout 600 python bench.py --config c3 --steps 5 > $O/bench_c3.json 2>/dev/null
timeout 600 python bench.py --config c4 --steps 5 > $O/bench_c4.json 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x -rs > $O/pytest_gpu.txt 2>&1
timeout 300 python bench.py --config c2 > $O/bench_c2.json 2>/dev/null
timeout 300 python bench.py --config c1 --graph --steps 20 > $O/bench_c1_graph.json 2>/dev/null
CMD3="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:hash_index -s 3 -c 1 -o $O/prof_c3 $CMD3 > $O/ncu_c3.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --collide-pairs 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launch.log 2>&1
echo done > $O/done.txt
