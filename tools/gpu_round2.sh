#!/bin/bash
set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gpu_parity.log 2>&1; tail -3 gpurun_out/gpu_parity.log
python tools/perf_probe.py > gpurun_out/perf.log 2>&1; tail -16 gpurun_out/perf.log
python bench.py --no-cpu --no-games > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 11 -c 1 -o gpurun_out/prof_bwd_n40 -f python tools/ncu_target.py 40 64 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
