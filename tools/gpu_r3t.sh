#!/bin/bash
mkdir -p gpurun_out
CFR_STREAM_EARLY=1 timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_variants.py tests/test_gpu_battleship.py -q -x -k "stream or streaming or fused" > gpurun_out/gpu_early_tests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/gpu_early_tests.log
AB_REPS=2 timeout 1200 python tools/ab_env.py 64 0 - CFR_STREAM_EARLY=1 > gpurun_out/ab_early2_64.log 2>&1; grep -A1 "rep 1" gpurun_out/ab_early2_64.log; grep SUMMARY gpurun_out/ab_early2_64.log
AB_REPS=2 timeout 1200 python tools/ab_env.py 32 0 - CFR_STREAM_EARLY=1 > gpurun_out/ab_early2_32.log 2>&1; grep SUMMARY gpurun_out/ab_early2_32.log
