mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bfgs.py -q -x -rA 2>&1 | tail -40 > gpurun_out/pytest_bfgs.txt
for a in "rosenbrock 50 16384 5" "rastrigin 50 65536 5" "ackley 50 65536 5"; do
  timeout 300 python scripts/phase_probe.py $a
  ZEUS_NO_WIDE=1 timeout 300 python scripts/phase_probe.py $a
done > gpurun_out/phase.txt 2>&1
cat gpurun_out/pytest_bfgs.txt gpurun_out/phase.txt
