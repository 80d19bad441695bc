set -x
mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? > gpurun_out/status11.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status11.txt
timeout 600 python bench.py > gpurun_out/b11_c2.log 2>&1; echo bench=$? >> gpurun_out/status11.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/b11_c1.log 2>&1
for c in c3 c4; do timeout 900 python bench.py --config $c --steps 3 --no-e2e --cpu-seconds 10 > gpurun_out/b11_${c}.log 2>&1; done
echo done >> gpurun_out/status11.txt
