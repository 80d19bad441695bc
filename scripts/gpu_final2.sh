mkdir -p gpurun_out/final2
python -c "from paper_1602_08393_b200 import build; build.build()"
for c in c3 c4 c2r; do timeout 900 python bench.py --config $c --steps 5 > gpurun_out/final2/bench_$c.json 2>/dev/null; done
echo done > gpurun_out/final2/status.txt
