#!/bin/bash
# A/B of the in-tree library against variants/lib_*.so (wide_ab.py), args: the wide_ab problem list
mkdir -p gpurun_out
for lib in paper_2603_28770_b200/libzeus_sm100.so variants/lib_*.so; do
  echo "== $lib"
  ZEUS_LIB=$lib timeout 900 python scripts/wide_ab.py "$@"
done 2>&1 | tee gpurun_out/ab.txt
