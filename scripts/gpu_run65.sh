mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "index or auto or e2e or hasher or sharding or maximum or key_space or csr" > gpurun_out/pytest_b65.log 2>&1; echo t=$? > gpurun_out/status65.txt
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
$B --config c3 > gpurun_out/b65_c3.log 2>&1
$B --config c4 > gpurun_out/b65_c4.log 2>&1
$B --config c2r > gpurun_out/b65_c2r.log 2>&1
echo done >> gpurun_out/status65.txt
