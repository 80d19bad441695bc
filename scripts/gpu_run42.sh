mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
python scripts/e2e_probe.py --bw > gpurun_out/e2e_8.json 2>&1
for c in 4 16 24 32 48; do WMH_E2E_CHUNKS=$c python scripts/e2e_probe.py > gpurun_out/e2e_$c.json 2>&1; done
echo done > gpurun_out/status42.txt
