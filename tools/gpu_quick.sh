#!/bin/bash
# quick loop: GPU tests, bench line (no cpu leg, no per-game), ncu launch list
set -x
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python bench.py --no-cpu --no-games --e2e-steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-games --no-cpu --e2e-steps 2 > gpurun_out/bench_ncu.json 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 22
