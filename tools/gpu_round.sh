#!/bin/bash
# one GPU session: bench line, ncu launch list, ncu full capture of the dominant kernel
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-games --no-cpu --e2e-steps 2 > gpurun_out/bench_ncu.json 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 11 -c 1 -o gpurun_out/prof_bwd_n40 -f python tools/ncu_target.py 40 64 2 > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/ncu_full.log
