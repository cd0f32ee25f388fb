#!/bin/bash
# One gpurun call: smoke, GPU tests, bench (c2 + north-star lines), ncu launch
# list of one c2 step, ncu --set full of the BFGS kernels (c2 tiers, T50b wide).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rA ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ -z "${NO_NCU:-}" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-north-star ${BENCH_ARGS:-} > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfgs_ -c 3 -o gpurun_out/prof_bfgs_c2 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-north-star ${BENCH_ARGS:-} > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfgs_wide -c 1 -o gpurun_out/prof_wide_t50b -f python bench.py --config t50b --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full_t50b.log 2>&1
fi
tail -3 gpurun_out/smoke.txt; tail -15 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
