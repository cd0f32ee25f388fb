mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bfgs.py tests/test_gpu_driver.py -q -x -rf 2>&1 | tail -5 > gpurun_out/pytest_thread.txt
for k in 8 12 16; do
  ZEUS_K1T=$k timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --no-north-star > gpurun_out/bench_thread_k$k.json 2>&1
done
timeout 300 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --no-north-star > gpurun_out/bench_thread_c1.json 2>&1
for a in "rastrigin 50 65536 5" "rosenbrock 50 16384 5"; do timeout 300 python scripts/phase_probe.py $a; done > gpurun_out/phase_thread.txt 2>&1
cat gpurun_out/pytest_thread.txt
for f in gpurun_out/bench_*thread*.json; do echo $f; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('  value %.4g ms/step %.3f bfgs %.3f launches %d' % (d['value'], d['ms_per_step'], d['bfgs_ms_per_step'], d['gpu_launches']))"; done
cat gpurun_out/phase_thread.txt
