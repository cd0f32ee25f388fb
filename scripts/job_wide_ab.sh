#!/bin/bash
# A/B of the wide kernel: SM-cycles per start-iteration (phase_probe) for the
# current library and variants/lib_*.so given as arguments; then its tests.
mkdir -p gpurun_out
for lib in paper_2603_28770_b200/libzeus_sm100.so "$@"; do
  for a in "rosenbrock 50 131072 5" "rastrigin 50 131072 5" "ackley 50 65536 5" "rosenbrock 100 16384 5"; do
    echo "$lib $a: $(ZEUS_LIB=$PWD/$lib timeout 300 python scripts/phase_probe.py $a 2>&1 | tail -1)"
  done
done > gpurun_out/wide_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bfgs.py -q -x 2>&1 | tail -3 >> gpurun_out/wide_ab.txt
cat gpurun_out/wide_ab.txt
