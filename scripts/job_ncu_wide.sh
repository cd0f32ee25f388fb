mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfgs_wide -c 1 -o gpurun_out/prof_wide_b50 -f python scripts/phase_probe.py rosenbrock 50 16384 5 > gpurun_out/ncu_wide1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfgs_wide -c 1 -o gpurun_out/prof_wide_r50 -f python scripts/phase_probe.py rastrigin 50 32768 5 > gpurun_out/ncu_wide2.log 2>&1
tail -2 gpurun_out/ncu_wide1.log gpurun_out/ncu_wide2.log
