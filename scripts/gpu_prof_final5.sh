O=gpurun_out/final5
mkdir -p $O
python -c "from paper_1602_08393_b200 import build; build.build()"
for c in c3 c4; do
CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $O/plain_$c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_index -s 3 -c 1 -o $O/prof_$c $CMD > $O/ncu_$c.log 2>&1
done
CMD="python bench.py --config c5 --gpu-gen --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $O/plain_c5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_tiled -s 3 -c 1 -o $O/prof_c5 $CMD > $O/ncu_c5.log 2>&1
echo done > $O/status.txt
