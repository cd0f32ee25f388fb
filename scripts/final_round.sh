#!/bin/bash
# Round-end evidence in one gpurun call: GPU tests, smoke, every bench config,
# the reference arm on T50, ncu launch lists + --set full captures of the
# T50 kernels and of the d = 20 / d = 100 kernels.
#   TAG=r02n bash scripts/final_round.sh
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rA > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench_t50.json 2> gpurun_out/${TAG}_bench_t50.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref_t50.json 2> gpurun_out/${TAG}_ref_t50.err
for c in c1 c2 c3 c4 c5; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 --no-python-reference > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
for c in t50b t50r; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_${c}_launches.csv python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-python-reference \
      > gpurun_out/${TAG}_${c}_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfgs_wide -c 1 \
      -o gpurun_out/${TAG}_${c} -f python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-python-reference \
      > gpurun_out/${TAG}_${c}_full.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfgs_wide -c 1 \
    -o gpurun_out/${TAG}_c4shard -f python scripts/wide_ab.py rosenbrock 100 131072 > gpurun_out/${TAG}_c4shard_full.log 2>&1
tail -3 gpurun_out/${TAG}_pytest_gpu.txt; cat gpurun_out/${TAG}_smoke.txt
