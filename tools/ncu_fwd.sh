#!/bin/bash
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 19 -c 1 -o gpurun_out/prof_fwd_n40 -f python tools/ncu_target.py 40 64 3 > gpurun_out/ncu_fwd.log 2>&1
tail -2 gpurun_out/ncu_fwd.log
