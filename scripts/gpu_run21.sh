mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m gpu -x -q -k "index or auto or u16" > gpurun_out/pytest_index.log 2>&1; echo pytest=$? > gpurun_out/status21.txt
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
export BENCH_CACHE_DIR=/tmp/bcache
for lm in 8 16 32 1000000; do WMH_INDEX_LMIN=$lm $B --config c3 > gpurun_out/b21_c3_l$lm.log 2>&1; done
for lm in 8 16 32 1000000; do WMH_INDEX_LMIN=$lm $B --config c4 > gpurun_out/b21_c4_l$lm.log 2>&1; done
for lm in 8 16 1000000; do WMH_INDEX_LMIN=$lm $B --algo index > gpurun_out/b21_c2_l$lm.log 2>&1; done
echo done >> gpurun_out/status21.txt
