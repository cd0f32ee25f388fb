mkdir -p gpurun_out
for a in "rosenbrock 50 16384 5" "rastrigin 50 65536 5" "ackley 50 65536 5" "rosenbrock 100 4096 5" "rastrigin 10 65536 20"; do
  ZEUS_LIB=$PWD/variants/lib_timing.so timeout 300 python scripts/phase_probe.py $a
done > gpurun_out/phase.txt 2>&1
cat gpurun_out/phase.txt
