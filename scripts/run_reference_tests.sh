#!/bin/bash
# Run the reference's own unit tests for the hot-path modules against this
# package (import shim tests/refshim: `import zeus` -> paper_2603_28770_b200).
#   here (build container):  bash scripts/run_reference_tests.sh stage
#     copies /root/reference/pkg/tests into the git-ignored baseline/_ref_tests
#   on the GPU box:          bash scripts/run_reference_tests.sh run
#     -> gpurun_out/reference_tests.txt (pytest -rA: every test's outcome)
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
case "${1:-run}" in
  stage)
    rm -rf "$ROOT/baseline/_ref_tests" && mkdir -p "$ROOT/baseline/_ref_tests"
    cp /root/reference/pkg/tests/test_{autodiff,objectives,linesearch,bfgs,pso,driver}.py \
       "$ROOT/baseline/_ref_tests/" ;;
  run)
    mkdir -p "$ROOT/gpurun_out"
    cd "$ROOT/baseline/_ref_tests" && PYTHONPATH="$ROOT/tests/refshim" \
      timeout 1800 python -m pytest -q -rA -p no:cacheprovider --rootdir . . \
      > "$ROOT/gpurun_out/reference_tests.txt" 2>&1
    tail -3 "$ROOT/gpurun_out/reference_tests.txt" ;;
esac
