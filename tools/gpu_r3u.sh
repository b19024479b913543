#!/bin/bash
mkdir -p gpurun_out
AB_REPS=2 timeout 900 python tools/ab_env.py 64 0 - > gpurun_out/ab_stagger_on.log 2>&1; grep SUMMARY gpurun_out/ab_stagger_on.log
CFR_B200_LIB_VARIANT=nostagger AB_REPS=2 timeout 900 python tools/ab_env.py 64 0 - > gpurun_out/ab_stagger_off.log 2>&1; grep SUMMARY gpurun_out/ab_stagger_off.log
AB_REPS=2 timeout 900 python tools/ab_env.py 64 0 - > gpurun_out/ab_stagger_on2.log 2>&1; grep SUMMARY gpurun_out/ab_stagger_on2.log
CFR_B200_LIB_VARIANT=nostagger AB_REPS=2 timeout 900 python tools/ab_env.py 32 0 - > gpurun_out/ab_stagger_off32.log 2>&1; grep SUMMARY gpurun_out/ab_stagger_off32.log
AB_REPS=2 timeout 900 python tools/ab_env.py 32 0 - > gpurun_out/ab_stagger_on32.log 2>&1; grep SUMMARY gpurun_out/ab_stagger_on32.log
