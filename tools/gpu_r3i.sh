#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_subtree.py -q -x > gpurun_out/gpu_sub_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_sub_tests.log
timeout 900 python tools/sub_ab.py leduc liars_dice goofspiel battleship3 > gpurun_out/sub_ab4.log 2>&1; cat gpurun_out/sub_ab4.log
timeout 600 python tools/sub_prof.py liars_dice goofspiel > gpurun_out/sub_prof2.log 2>&1; cat gpurun_out/sub_prof2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sub<" -s 3 -c 1 -o gpurun_out/prof_ksub_liars -f python tools/ncu_sub_target.py liars_dice 5 > gpurun_out/ncu_sub.log 2>&1; tail -2 gpurun_out/ncu_sub.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_liars.csv python tools/ncu_sub_target.py liars_dice 5 > /dev/null 2>&1; tail -8 gpurun_out/launches_liars.csv
