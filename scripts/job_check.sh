mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -rf ${PYTEST_ARGS:-} 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
[ -z "${NO_BENCH:-}" ] && timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/pytest_gpu.txt gpurun_out/bench.json 2>/dev/null; tail -3 gpurun_out/bench.err 2>/dev/null
