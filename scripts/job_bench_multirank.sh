#!/bin/bash
# bench.py's N > 1 path on a one-GPU box: 2 ranks over gloo on GPU 0, with
# the collective barrier and with the peer-memory exchange (IPC)
mkdir -p gpurun_out
for ex in collective peer; do
  ZEUS_BENCH_DEVICE=0 ZEUS_BENCH_BACKEND=gloo ZEUS_PSO_EXCHANGE=$ex timeout 600 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --steps 2 --warmup 3 \
    --no-cpu-baseline --no-north-star > gpurun_out/bench_mr_$ex.json 2> gpurun_out/bench_mr_$ex.err
  echo "$ex rc=$?"; head -c 600 gpurun_out/bench_mr_$ex.json; echo; tail -3 gpurun_out/bench_mr_$ex.err
done
