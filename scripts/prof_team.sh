mkdir -p gpurun_out
timeout 300 python scripts/latency_probe.py rastrigin 50 16384 5 > gpurun_out/probe_r50.txt 2>&1
timeout 300 python scripts/latency_probe.py rosenbrock 100 2048 5 > gpurun_out/probe_b100.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfgs_team -c 1 -o gpurun_out/prof_team_r50 -f python bench.py --config t50r --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/probe_r50.txt gpurun_out/probe_b100.txt
