mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfgs_thread -c 1 -o gpurun_out/prof_thread_r10 -f python scripts/phase_probe.py rastrigin 10 65536 20 > gpurun_out/ncu_thread.log 2>&1
tail -2 gpurun_out/ncu_thread.log
