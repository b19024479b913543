#!/bin/bash
# full GPU suite, smoke, default bench (with per-config lines), sanitizers
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --durations=20 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
bash tools/gpu_sanitize.sh
