#!/bin/bash
# GPU test pass on the box: pytest -m gpu (+ optional -k filter in $1), smoke
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then
  timeout 3000 python -m pytest tests -q -m gpu -k "$K" -x --durations=15 > gpurun_out/gpu_tests.log 2>&1
else
  timeout 3000 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/gpu_tests.log 2>&1
fi
echo "pytest rc=$?"
tail -45 gpurun_out/gpu_tests.log
