set -x
mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
for c in c3 c4; do for ch in 1000 3000 8000; do
CMD="python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 3 --config $c --rows 16384 --algo index"
WMH_INDEX_CHUNKS=$ch $CMD > /dev/null 2>&1 && WMH_INDEX_CHUNKS=$ch ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches10_${c}_$ch.csv $CMD > /dev/null 2>&1
done; done
echo done > gpurun_out/status10.txt
