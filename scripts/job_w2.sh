mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bfgs.py -q -x -rf --timeout 600 2>&1 | tail -12
for a in "rosenbrock 100 4096 5" "rastrigin 100 16384 5" "ackley 100 16384 5"; do
  timeout 300 python scripts/phase_probe.py $a; ZEUS_NO_WIDE=1 timeout 300 python scripts/phase_probe.py $a
done 2>&1 | python -c "
import sys, json
for line in sys.stdin:
    try: d = json.loads(line); print(d['objective'], d['d'], 'bfgs_ms %.2f sm_cyc/start-iter %.0f' % (d['bfgs_ms'], d['sm_cycles_per_start_iter']))
    except Exception: print(line.rstrip()[:200])"
