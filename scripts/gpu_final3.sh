mkdir -p gpurun_out/final3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final3/build.log 2>&1; echo build=$? > gpurun_out/final3/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3/smoke.log 2>&1; echo smoke=$? >> gpurun_out/final3/status.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final3/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/final3/status.txt
timeout 600 python bench.py > gpurun_out/final3/bench_c2.json 2>/dev/null; echo bench=$? >> gpurun_out/final3/status.txt
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final3/launches_c2.csv $CMD > /dev/null 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hash_tiled_cm -s 3 -c 1 -o gpurun_out/final3/prof_c2_cm $CMD > /dev/null 2>&1
timeout 1200 python bench.py --config c5 --gpu-gen --steps 3 --collide-pairs 10000000 > gpurun_out/final3/bench_c5.json 2>/dev/null
echo done >> gpurun_out/final3/status.txt
