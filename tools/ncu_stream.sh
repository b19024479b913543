#!/bin/bash
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bwd_stream -s 12 -c 1 -o gpurun_out/prof_stream_n40 -f python tools/ncu_target.py 40 64 4 > gpurun_out/ncu_stream.log 2>&1
tail -3 gpurun_out/ncu_stream.log
