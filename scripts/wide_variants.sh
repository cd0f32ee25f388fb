#!/bin/bash
# Build libzeus variants that differ only in bfgs_wide.cu's tuning macros:
#   scripts/wide_variants.sh NAME "-DZEUS_WIDE_RR_OVERRIDE=24 -DZEUS_WIDE_MINB=4 -DZEUS_WIDE_CH=4" ...
# (pairs of name + flags); outputs variants/lib_<name>.so
set -e
cd "$(dirname "$0")/.."
C=paper_2603_28770_b200/csrc
make -s -C $C -j6 >/dev/null
mkdir -p variants
FL="-O3 -std=c++17 -lineinfo -fmad=false -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
OTHERS=$(ls $C/build/*.o | grep -v bfgs_wide.o)
pids=()
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ( mkdir -p /tmp/wv_$name
    nvcc $FL $flags -c $C/bfgs_wide.cu -o /tmp/wv_$name/bfgs_wide.o 2> /tmp/wv_$name/ptxas.log
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$name.so /tmp/wv_$name/bfgs_wide.o $OTHERS -lcudart -lnvrtc
    echo "$name: $(grep -A2 'bfgs_wide_kernel' /tmp/wv_$name/ptxas.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' ')" ) &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
