mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_real.py -m gpu -x -q -k "index or auto or u16 or e2e or hasher or sharding or edge" > gpurun_out/pytest_b48.log 2>&1; echo t=$? > gpurun_out/status48.txt
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
$B --config c4 > gpurun_out/b48_c4.log 2>&1
$B --config c3 > gpurun_out/b48_c3.log 2>&1
$B --config c2r > gpurun_out/b48_c2r.log 2>&1
CMD="python bench.py --config c5 --gpu-gen --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_tiled -s 3 -c 1 -o gpurun_out/prof_c5_bs $CMD > gpurun_out/ncu_c5_bs.log 2>&1
echo done >> gpurun_out/status48.txt
