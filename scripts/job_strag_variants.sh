for lib in paper_2603_28770_b200/libzeus_sm100.so variants/lib_*.so; do
  echo "$lib $(ZEUS_LIB=$PWD/$lib timeout 300 python scripts/latency_probe.py 2>&1 | tail -1 | python -c "
import sys, json; d = json.loads(sys.stdin.read()); print('straggler cycles/iter %.0f' % d['cycles_per_iteration_at_1965MHz'])") | $(ZEUS_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-north-star 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2 ms/step %.2f bfgs %.2f' % (d['ms_per_step'], d['bfgs_ms_per_step']))")"
done
