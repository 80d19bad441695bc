mkdir -p gpurun_out/final
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 600 python bench.py > gpurun_out/final/bench_c2.json 2>gpurun_out/final/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_c2_reference.json 2>/dev/null
timeout 300 python bench.py --config c1 > gpurun_out/final/bench_c1.json 2>/dev/null
timeout 600 python bench.py --config c2r > gpurun_out/final/bench_c2r.json 2>/dev/null
timeout 900 python bench.py --config c3 --steps 5 > gpurun_out/final/bench_c3.json 2>/dev/null
timeout 900 python bench.py --config c4 --steps 5 > gpurun_out/final/bench_c4.json 2>/dev/null
timeout 1200 python bench.py --config c5 --gpu-gen --steps 3 --collide-pairs 10000000 > gpurun_out/final/bench_c5.json 2>/dev/null
echo done > gpurun_out/final/status.txt
