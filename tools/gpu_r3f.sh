#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/sub_cut_sweep.py leduc liars_dice goofspiel battleship2 battleship3 battleship4 battleship5 > gpurun_out/sub_cut.log 2>&1; cat gpurun_out/sub_cut.log | tail -20
timeout 2400 python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/gpu_tests.log
