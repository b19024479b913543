#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -k "parity or variants or errors or br or c_program" > gpurun_out/gpu_tiny_tests.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/gpu_tiny_tests.log
timeout 600 python tools/perf_probe.py > gpurun_out/perf.log 2>&1; echo "perf rc=$?"; cat gpurun_out/perf.log | cut -c1-140
