mkdir -p gpurun_out
( ZEUS_LIB=$PWD/variants/lib_timing.so timeout 300 python scripts/latency_probe.py
  timeout 300 python scripts/latency_probe.py
  ZEUS_K1=0 timeout 300 python scripts/latency_probe.py ) > gpurun_out/lat.txt 2>&1
cat gpurun_out/lat.txt
