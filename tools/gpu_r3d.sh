#!/bin/bash
# fused forward + L2-prefetch warp: parity tests of the fused path, then A/B fused vs separate forward
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "fused or stream_synthetic" > gpurun_out/gpu_fused_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_fused_tests.log
timeout 900 python tools/stream_cfg_sweep.py 64 2:0:0 2:0:64 2:0:0 2:0:64 > gpurun_out/sweep_fused64.log 2>&1; grep "cfg=" gpurun_out/sweep_fused64.log
timeout 900 python tools/stream_cfg_sweep.py 32 2:0:0 2:0:64 2:0:0 2:0:64 > gpurun_out/sweep_fused32.log 2>&1; grep "cfg=" gpurun_out/sweep_fused32.log
