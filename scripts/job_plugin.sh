mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_plugin.py tests/test_harness.py tests/test_gpu_bfgs.py -q -x -rf --timeout 600 2>&1 | tail -30 > gpurun_out/pytest_plugin.txt
cat gpurun_out/pytest_plugin.txt
