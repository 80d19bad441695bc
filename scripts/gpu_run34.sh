mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
for cf in 16 48 128; do WMH_INDEX_CF=$cf $B --config c4 > gpurun_out/b34_c4_cf$cf.log 2>&1; done
echo done >> gpurun_out/status34.txt
