#!/bin/bash
# Final-state ncu evidence (one gpurun call): launch lists + --set full of the
# BFGS kernel for T50 (each problem alone), config 3, config 5's largest grid
# point, and config 4's 131,072-start shard (the 1M-start capture exceeds the
# replay budget).   TAG=r02i bash scripts/profile_final.sh
TAG=${TAG:-r02}
mkdir -p gpurun_out
for cfg in t50b t50r c3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_${cfg}_launches.csv python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline --no-python-reference \
      > gpurun_out/${TAG}_${cfg}_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfgs_wide -c 1 \
      -o gpurun_out/${TAG}_${cfg} -f python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline --no-python-reference \
      > gpurun_out/${TAG}_${cfg}_full.log 2>&1
  echo "$cfg rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfgs_wide -c 1 \
    -o gpurun_out/${TAG}_c4shard -f python scripts/wide_ab.py rosenbrock 100 131072 \
    > gpurun_out/${TAG}_c4shard_full.log 2>&1
echo "c4shard rc=$?"
