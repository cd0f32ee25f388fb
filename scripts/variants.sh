#!/bin/bash
# probe + C2 bench per library variant (ZEUS_LIB override)
mkdir -p gpurun_out
for lib in paper_2603_28770_b200/libzeus_sm100.so variants/*.so; do
  echo "== $lib"
  ZEUS_LIB=$PWD/$lib timeout 300 python scripts/latency_probe.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  straggler us/iter %.2f cycles %.0f' % (d['us_per_iteration'], d['cycles_per_iteration_at_1965MHz']))"
  ZEUS_LIB=$PWD/$lib timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  c2 ms/step %.2f bfgs %.2f value %.3g' % (d['ms_per_step'], d['bfgs_ms_per_step'], d['value']))"
done
