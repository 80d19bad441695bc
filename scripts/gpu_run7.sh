set -x
mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "index" > gpurun_out/pytest_index.log 2>&1; echo pytest=$? > gpurun_out/status7.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 --algo index"
for cf in 0.25 0.5 1 2; do WMH_INDEX_CF=$cf $B > gpurun_out/b7_c2_cf$cf.log 2>&1; done
WMH_INDEX_NW=4 $B > gpurun_out/b7_c2_nw4.log 2>&1
for cf in 0.25 0.5 1 2; do WMH_INDEX_CF=$cf $B --config c5 --rows 262144 --gpu-gen > gpurun_out/b7_c5_cf$cf.log 2>&1; done
for c in c3 c4; do $B --config $c > gpurun_out/b7_${c}_full.log 2>&1; done
echo done >> gpurun_out/status7.txt
