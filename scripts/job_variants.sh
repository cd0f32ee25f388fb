# phase_probe for each variants/lib_*.so on the d=50 objectives (+ parity of the default lib)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_bfgs.py -q -x 2>&1 | tail -2
for lib in paper_2603_28770_b200/libzeus_sm100.so variants/lib_*.so; do
  for a in ${PROBES:-"rosenbrock 50 16384 5" "rastrigin 50 65536 5"}; do
    echo "$lib $a $(ZEUS_LIB=$PWD/$lib timeout 120 python scripts/phase_probe.py $a 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("bfgs_ms %.2f sm_cyc/start-iter %.0f" % (d["bfgs_ms"], d["sm_cycles_per_start_iter"]))' 2>&1)"
  done
done 2>&1 | tee gpurun_out/variants.txt
