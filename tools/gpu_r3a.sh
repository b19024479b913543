#!/bin/bash
# evidence on HEAD: full GPU suite, smoke, default bench
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; head -c 1500 gpurun_out/bench.json
