#!/bin/bash
# ncu evidence for the bench configurations (one gpurun call): per config the
# launch list of one bench.py step and --set full captures of its BFGS kernels.
#   TAG=r02b bash scripts/profile_r02.sh [config ...]
TAG=${TAG:-r02}
mkdir -p gpurun_out
for cfg in ${@:-t50 c3 c4 c5s}; do
  args="--config $cfg --steps 1 --warmup 0 --no-cpu-baseline"
  case $cfg in
    c5s) args="--config c5 --steps 1 --warmup 0 --no-cpu-baseline"; kfilter="regex:bfgs_warp"; cnt=1;
         # the 1M-start, 20-sweep, cap-1024 grid point: launch 54 (0-based 53) of the grid's BFGS kernels
         skip="--launch-skip 53";;
    t50) kfilter="regex:bfgs_wide"; cnt=2; skip="";;
    *) kfilter="regex:bfgs_"; cnt=3; skip="";;
  esac
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_${cfg}_launches.csv python bench.py $args \
      > gpurun_out/${TAG}_${cfg}_launch.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k $kfilter $skip -c $cnt \
      -o gpurun_out/${TAG}_${cfg} -f python bench.py $args > gpurun_out/${TAG}_${cfg}_full.log 2>&1
  echo "$cfg done rc=$?"
done
