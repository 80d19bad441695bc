mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bitplanes or (parity_configs and tiled)" > gpurun_out/pytest_b39.log 2>&1; echo t=$? > gpurun_out/status39.txt
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
$B --config c2 --algo tiled > gpurun_out/b39_c2_bs.log 2>&1
$B --config c5 --rows 1000000 --gpu-gen --algo tiled > gpurun_out/b39_c5_bs.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_tiled_bs -s 3 -c 1 -o gpurun_out/prof_c2_bs2 $CMD > gpurun_out/ncu_c2_bs2.log 2>&1
echo done >> gpurun_out/status39.txt
