#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/stream_cfg_sweep.py 64 2:0:0 2:0:0 > gpurun_out/sweep_hint.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep_hint.log
timeout 900 python -m pytest tests -q -m gpu -x -k "stream or bench_shaped or sharded" > gpurun_out/gpu_stream_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_stream_tests.log
