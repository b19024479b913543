#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_subtree.py -q -x -k "band" > gpurun_out/gpu_band_tests.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gpu_band_tests.log
AB_REPS=2 timeout 1200 python tools/ab_env.py 64 0 - CFR_BAND=0 > gpurun_out/ab_band64.log 2>&1; grep -A1 "rep 1" gpurun_out/ab_band64.log; grep SUMMARY gpurun_out/ab_band64.log
AB_REPS=2 timeout 1200 python tools/ab_env.py 32 0 - CFR_BAND=0 > gpurun_out/ab_band32.log 2>&1; grep SUMMARY gpurun_out/ab_band32.log
