#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_subtree.py tests/test_gpu_errors.py tests/test_gpu_resume.py tests/test_gpu_parity_configs.py -q -x -k "not sharded" > gpurun_out/gpu_trunk_tests.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gpu_trunk_tests.log
timeout 600 python tools/sub_ab.py leduc liars_dice > gpurun_out/sub_ab_trunk.log 2>&1; cat gpurun_out/sub_ab_trunk.log
CFR_SUB_TRUNK=0 timeout 600 python tools/sub_ab.py leduc liars_dice > gpurun_out/sub_ab_notrunk.log 2>&1; cat gpurun_out/sub_ab_notrunk.log
