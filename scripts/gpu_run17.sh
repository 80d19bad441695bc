mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 600 python bench.py --config c2r > gpurun_out/b17_c2r.log 2>&1; echo c2r=$? > gpurun_out/status17.txt
timeout 600 python bench.py --config c2r --algo simple --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/b17_c2r_simple.log 2>&1
timeout 600 python bench.py --config c5 --gpu-gen --rows 1000000 --steps 3 --no-e2e > gpurun_out/b17_c5_1m.log 2>&1; echo c5=$? >> gpurun_out/status17.txt
