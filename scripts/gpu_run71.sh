mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_b71.log 2>&1; echo t=$? > gpurun_out/status71.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke71.log 2>&1; echo smoke=$? >> gpurun_out/status71.txt
O=gpurun_out/final10; mkdir -p $O
timeout 1200 python bench.py --config c5 --gpu-gen --steps 3 --collide-pairs 10000000 > $O/bench_c5.json 2>/dev/null
CMD="python bench.py --config c5 --gpu-gen --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_tiled -s 3 -c 1 -o $O/prof_c5 $CMD > $O/ncu_c5.log 2>&1
echo done >> gpurun_out/status71.txt
