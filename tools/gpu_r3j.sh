#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:^k_sub$ -s 3 -c 1 -o gpurun_out/prof_ksub_liars -f python tools/ncu_sub_target.py liars_dice 5 > gpurun_out/ncu_sub.log 2>&1; tail -3 gpurun_out/ncu_sub.log
