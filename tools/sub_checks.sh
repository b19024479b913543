#!/bin/bash
# Bounds-checked subtree kernels (-DCFR_SUB_CHECKS: trap on any out-of-range table
# entry or shared-memory index) through the subtree parity tests; compute-sanitizer
# is closed on this pool.  Builds libcfr_b200.checks.so next to the product library.
mkdir -p gpurun_out
python -c "from paper_2408_14778_b200 import _native; _native.build(variant='checks', defines=['CFR_SUB_CHECKS'])" || exit 1
CFR_B200_LIB_VARIANT=checks timeout 1500 python -m pytest tests/test_gpu_subtree.py tests/test_gpu_parity_configs.py -q -x -k "subtree or liars or goofspiel or leduc" > gpurun_out/sub_checks.log 2>&1
echo "checked run rc=$?"; tail -3 gpurun_out/sub_checks.log
