#!/bin/bash
# subtree mode: parity tests, then per-game A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_subtree.py -q -x > gpurun_out/gpu_sub_tests.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/gpu_sub_tests.log
timeout 900 python tools/sub_ab.py > gpurun_out/sub_ab.log 2>&1; cat gpurun_out/sub_ab.log | tail -40
