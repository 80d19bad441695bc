mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
WMH_E2E_TRACE=1 python scripts/e2e_probe.py > gpurun_out/e2e_trace_b.log 2>&1
WMH_E2E_TRACE=1 WMH_E2E_CHUNKS=8 python scripts/e2e_probe.py > gpurun_out/e2e_trace8_b.log 2>&1
WMH_E2E_TRACE=1 WMH_E2E_CHUNKS=6 python scripts/e2e_probe.py > gpurun_out/e2e_trace6_b.log 2>&1
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
$B --config c2 > gpurun_out/b45_c2.log 2>&1
for r in 3300 13300; do for m in 16 32 64 128; do WMH_MIN_HCHUNK=$m $B --config c2 --rows $r > gpurun_out/b45_c2_${r}_$m.log 2>&1; done; done
echo done > gpurun_out/status45.txt
