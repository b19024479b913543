#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_subtree.py -q -x -k "deferred or liars or real_games" > gpurun_out/gpu_sub_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_sub_tests.log
timeout 900 python tools/sub_ab.py goofspiel6 > gpurun_out/sub_ab8.log 2>&1; cat gpurun_out/sub_ab8.log
timeout 900 python tools/sub_cut_sweep.py goofspiel6 > gpurun_out/sub_cut4.log 2>&1; cat gpurun_out/sub_cut4.log
