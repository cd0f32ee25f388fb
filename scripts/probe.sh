mkdir -p gpurun_out
timeout 300 python scripts/latency_probe.py > gpurun_out/probe.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfgs_warp -s 2 -c 1 -o gpurun_out/prof_straggler -f python scripts/latency_probe.py > gpurun_out/ncu_probe.log 2>&1
cat gpurun_out/probe.txt; tail -3 gpurun_out/ncu_probe.log
