set -x
mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
for c in c4 c3; do
CMD="python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 3 --config $c --rows 16384 --algo index"
$CMD > gpurun_out/plain_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hash_index -s 3 -c 1 -o gpurun_out/prof_index_$c $CMD > gpurun_out/ncu_$c.log 2>&1
done
