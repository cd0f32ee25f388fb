# usage: PROBES="rosenbrock:50:16384:5 rastrigin:50:65536:5" bash scripts/job_wide_check.sh
for lib in paper_2603_28770_b200/libzeus_sm100.so variants/lib_*.so; do
  for a in ${PROBES:-rosenbrock:50:16384:5}; do
    echo "$lib $(ZEUS_LIB=$PWD/$lib timeout 300 python scripts/phase_probe.py ${a//:/ } 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print(d['objective'], d['d'], 'bfgs_ms %.2f sm_cyc/start-iter %.0f' % (d['bfgs_ms'], d['sm_cycles_per_start_iter']))")"
  done
done
