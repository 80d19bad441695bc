mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m gpu -x -q -k "index or auto or u16 or e2e" > gpurun_out/pytest_index.log 2>&1; echo pytest=$? > gpurun_out/status29.txt
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
for o in 1 0; do WMH_INDEX_ORDER=$o $B --config c4 > gpurun_out/b29_c4_o$o.log 2>&1; done
for o in 1 0; do WMH_INDEX_ORDER=$o $B --config c3 > gpurun_out/b29_c3_o$o.log 2>&1; done
for o in 1 0; do WMH_INDEX_ORDER=$o $B --config c2r > gpurun_out/b29_c2r_o$o.log 2>&1; done
echo done >> gpurun_out/status29.txt
