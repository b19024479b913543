#!/bin/bash
# round-end evidence on HEAD: GPU suite, smoke, default bench, reference arm, ncu launch
# list of one bench run, ncu --set full of the dominant launch (k_bwd_stream, level 10)
# and of k_sub (liar's dice)
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; head -c 600 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; head -c 400 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-games --no-cpu --e2e-steps 2 > gpurun_out/bench_ncu.json 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 22 > gpurun_out/launches_summary.txt; cat gpurun_out/launches_summary.txt | head -30
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bwd_stream -s 12 -c 1 -o gpurun_out/prof_stream_n40 -f python tools/ncu_target.py 40 64 4 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:^k_sub$ -s 3 -c 1 -o gpurun_out/prof_sub_liars -f python tools/ncu_sub_target.py liars_dice 5 > gpurun_out/ncu_sub.log 2>&1; tail -2 gpurun_out/ncu_sub.log
