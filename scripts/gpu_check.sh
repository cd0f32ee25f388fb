#!/bin/bash
# One gpurun call: smoke, GPU tests, the bench line (T50 headline) and the
# reference arm, then (unless NO_NCU) ncu evidence via profile_r02.sh.
#   TAG=r02b PROFILE_CONFIGS="t50 c3" bash scripts/gpu_check.sh
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
if [ -z "${NO_TESTS:-}" ]; then
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rA --durations=25 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
if [ -z "${NO_REF:-}" ]; then
timeout 900 python bench.py --impl reference ${BENCH_ARGS:-} > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?" >> gpurun_out/${TAG}_ref.err
fi
if [ -z "${NO_NCU:-}" ]; then
TAG=$TAG bash scripts/profile_r02.sh ${PROFILE_CONFIGS:-t50}
fi
tail -3 gpurun_out/smoke.txt; tail -40 gpurun_out/pytest_gpu.txt; cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_ref.json
