mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_b64.log 2>&1; echo t=$? > gpurun_out/status64.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke64.log 2>&1; echo smoke=$? >> gpurun_out/status64.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b64_c2.json 2>/dev/null; echo bench=$? >> gpurun_out/status64.txt
