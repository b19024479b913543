#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/gpu_stream.log 2>&1; tail -30 gpurun_out/gpu_stream.log
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu --no-games --e2e-steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-games --no-cpu --e2e-steps 2 > gpurun_out/bench_ncu.json 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 22
