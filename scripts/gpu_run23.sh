mkdir -p gpurun_out
python -c "from paper_1602_08393_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_fig2.py -m gpu -q > gpurun_out/pytest_fig2.log 2>&1; echo fig2=$? > gpurun_out/status23.txt
python scripts/fig2_accuracy.py gpurun_out/fig2_accuracy.csv > gpurun_out/fig2.log 2>&1
