#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_subtree.py -q -x > gpurun_out/gpu_sub_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gpu_sub_tests.log
timeout 900 python tools/sub_ab.py leduc liars_dice goofspiel battleship3 battleship5 > gpurun_out/sub_ab6.log 2>&1; cat gpurun_out/sub_ab6.log
