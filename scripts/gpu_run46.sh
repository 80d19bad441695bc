mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
for i in 1 2; do python scripts/e2e_probe.py > gpurun_out/e2e_r$i.json 2>&1; WMH_E2E_CHUNKS=8 python scripts/e2e_probe.py > gpurun_out/e2e_u$i.json 2>&1; WMH_E2E_CHUNKS=12 python scripts/e2e_probe.py > gpurun_out/e2e_v$i.json 2>&1; done
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
for r in 3300 13300; do for m in 256 512; do WMH_MIN_HCHUNK=$m $B --config c2 --rows $r > gpurun_out/b46_c2_${r}_$m.log 2>&1; done; done
$B --config c2 > gpurun_out/b46_c2.log 2>&1
echo done > gpurun_out/status46.txt
