#!/bin/bash
# evidence: Fig 3 curves, ncu launch list of one bench iteration
mkdir -p gpurun_out
timeout 900 python tools/fig3_curves.py > gpurun_out/fig3.log 2>&1; echo "fig3 rc=$?"; cat gpurun_out/fig3.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-games --no-cpu --no-variants --e2e-steps 2 > gpurun_out/bench_ncu.json 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches.csv 22 > gpurun_out/launches_summary.txt; tail -25 gpurun_out/launches_summary.txt
