mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
WMH_E2E_TRACE=1 python scripts/e2e_probe.py > gpurun_out/e2e_trace.log 2>&1
WMH_E2E_TRACE=1 WMH_E2E_CHUNKS=8 python scripts/e2e_probe.py > gpurun_out/e2e_trace8.log 2>&1
echo done > gpurun_out/status44.txt
