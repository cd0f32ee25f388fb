mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfgs_warp_kernel -s 3 -c 1 -o gpurun_out/prof_straggler -f python scripts/latency_probe.py > gpurun_out/ncu_strag.log 2>&1
tail -3 gpurun_out/ncu_strag.log
