mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_lsh.py -m gpu -q > gpurun_out/pytest_lsh.log 2>&1; echo lsh=$? > gpurun_out/status28.txt
timeout 600 python scripts/lsh_bench.py > gpurun_out/lsh_bench.json 2> gpurun_out/lsh_bench.err
