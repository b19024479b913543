#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_subtree.py tests/test_gpu_errors.py tests/test_gpu_resume.py tests/test_gpu_parity_configs.py tests/test_gpu_battleship.py tests/test_gpu_variants.py tests/test_gpu_parity.py -q -x -k "not sharded" > gpurun_out/gpu_trunk2_tests.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gpu_trunk2_tests.log
timeout 900 python tools/sub_ab.py leduc liars_dice goofspiel battleship3 battleship5 > gpurun_out/sub_ab_trunk2.log 2>&1; cat gpurun_out/sub_ab_trunk2.log
