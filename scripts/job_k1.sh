for k1 in 32 48 64 96; do for k1t in 16; do
  echo "k1=$k1 k1t=$k1t $(ZEUS_K1=$k1 ZEUS_K1T=$k1t timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-north-star 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c2 ms/step %.2f bfgs %.2f' % (d['ms_per_step'], d['bfgs_ms_per_step']))")"
done; done
