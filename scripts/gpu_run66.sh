mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
$B --config c3 > gpurun_out/b66_c3_head.log 2>&1
$B --config c4 > gpurun_out/b66_c4_head.log 2>&1
cp paper_1602_08393_b200/csrc/hash_index.cu.new paper_1602_08393_b200/csrc/hash_index.cu
python -c "from paper_1602_08393_b200 import build; build.build(force=True)"
$B --config c3 > gpurun_out/b66_c3_new.log 2>&1
$B --config c4 > gpurun_out/b66_c4_new.log 2>&1
$B --config c3 > gpurun_out/b66_c3_new2.log 2>&1
echo done > gpurun_out/status66.txt
