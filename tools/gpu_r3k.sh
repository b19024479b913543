#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_subtree.py -q -x > gpurun_out/gpu_sub_tests.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gpu_sub_tests.log
timeout 900 python tools/sub_cut_sweep.py leduc liars_dice goofspiel battleship2 battleship3 battleship4 battleship5 > gpurun_out/sub_cut2.log 2>&1; cat gpurun_out/sub_cut2.log | tail -20
timeout 900 python tools/sub_ab.py leduc liars_dice goofspiel battleship3 battleship5 battleship7 > gpurun_out/sub_ab5.log 2>&1; cat gpurun_out/sub_ab5.log
