#!/bin/bash
# quick per-config bench lines (no CPU baseline)
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c1 c3 t50r t50b c4}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-north-star > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json'))
print('  $c', d['config']['workload'], '| value %.4g starts/s | ms/step %.2f | bfgs %.2f ms | frac %.4f | achieved %.3f TF | generic %.3f TF' % (d['value'], d['ms_per_step'], d['bfgs_ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'], d['roofline']['achieved_generic_convention']))" 2>/dev/null || tail -3 gpurun_out/bench_$c.err
done
