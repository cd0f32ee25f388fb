#!/bin/bash
# libzeus variants differing only in bfgs.cu's macros: NAME "FLAGS" ...
set -e
cd "$(dirname "$0")/.."
C=paper_2603_28770_b200/csrc
make -s -C $C -j6 >/dev/null
mkdir -p variants
FL="-O3 -std=c++17 -lineinfo -fmad=false -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
OTHERS=$(ls $C/build/*.o | grep -v "/bfgs.o")
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ( mkdir -p /tmp/bv_$name
    nvcc $FL $flags -c $C/bfgs.cu -o /tmp/bv_$name/bfgs.o 2> /tmp/bv_$name/ptxas.log
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$name.so /tmp/bv_$name/bfgs.o $OTHERS -lcudart -lnvrtc ) &
done
wait
ls variants
