#!/bin/bash
# Build the product library (+ optional diagnostic variants); fails loudly.
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2603_28770_b200/csrc -j6
if [ -n "${TIMING:-}" ]; then
  mkdir -p variants
  make -s -C paper_2603_28770_b200/csrc -j6 BUILD=/tmp/bv_timing OUT=$PWD/variants/lib_timing.so EXTRA="-DZEUS_PHASE_TIMING"
fi
ls -la --time-style=+%T paper_2603_28770_b200/libzeus_sm100.so ${TIMING:+variants/lib_timing.so} | awk '{print "built", $6, $7}'
