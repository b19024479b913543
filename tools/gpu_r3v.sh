#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_variants.py -q -x -k "stream or streaming" > gpurun_out/gpu_pred_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_pred_tests.log
AB_REPS=3 timeout 900 python tools/ab_env.py 64 0 - > gpurun_out/ab_pred64.log 2>&1; grep SUMMARY gpurun_out/ab_pred64.log
AB_REPS=2 timeout 900 python tools/ab_env.py 64 0 CFR_STREAM_LATE_RELEASE=0 > gpurun_out/ab_pred64b.log 2>&1; grep SUMMARY gpurun_out/ab_pred64b.log
