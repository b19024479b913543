#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x -k "two_level or stream_synthetic" > gpurun_out/gpu_fwd2_tests.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gpu_fwd2_tests.log
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -k "streaming" > gpurun_out/gpu_fwd2_var.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_fwd2_var.log
AB_REPS=2 timeout 1200 python tools/ab_env.py 64 0 - CFR_FWD2=0 > gpurun_out/ab_fwd2_64.log 2>&1; grep -A1 "rep 1" gpurun_out/ab_fwd2_64.log; grep SUMMARY gpurun_out/ab_fwd2_64.log
AB_REPS=2 timeout 1200 python tools/ab_env.py 32 0 - CFR_FWD2=0 > gpurun_out/ab_fwd2_32.log 2>&1; grep SUMMARY gpurun_out/ab_fwd2_32.log
