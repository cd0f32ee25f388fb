for lib in variants/lib_timing.so variants/lib_timing4.so; do echo "== $lib"; ZEUS_LIB=$PWD/$lib timeout 300 python scripts/latency_probe.py 2>&1 | tail -4; done
ZEUS_LIB=$PWD/variants/lib_timing.so timeout 300 python scripts/latency_probe.py rosenbrock 50 4096 5 2>&1 | tail -4
