mkdir -p gpurun_out/check
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/check/build.log 2>&1; echo build=$? > gpurun_out/check/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check/smoke.log 2>&1; echo smoke=$? >> gpurun_out/check/status.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/check/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/check/status.txt
timeout 600 python bench.py > gpurun_out/check/bench.json 2> gpurun_out/check/bench.err; echo bench=$? >> gpurun_out/check/status.txt
