set -x
mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "index" > gpurun_out/pytest_index.log 2>&1; echo pytest=$? >> gpurun_out/status2.txt
B="timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
for a in tiled index; do WMH_INDEX_STATS=1 $B --algo $a > gpurun_out/b2_c2_$a.log 2>&1; done
for c in c3 c4; do for a in tiled index; do WMH_INDEX_STATS=1 $B --config $c --rows 16384 --algo $a > gpurun_out/b2_${c}_$a.log 2>&1; done; done
for a in tiled index; do WMH_INDEX_STATS=1 $B --config c5 --rows 262144 --gpu-gen --algo $a > gpurun_out/b2_c5_$a.log 2>&1; done
echo done >> gpurun_out/status2.txt
