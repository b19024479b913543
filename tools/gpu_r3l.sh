#!/bin/bash
mkdir -p gpurun_out
AB_REPS=2 timeout 1200 python tools/ab_env.py 64 0 - CFR_STREAM_MIN_TILES=400 CFR_STREAM_MIN_TILES=1200 CFR_STREAM_MIN_TILES=4000 > gpurun_out/ab_mintiles.log 2>&1; grep -A1 "rep 1" gpurun_out/ab_mintiles.log; grep SUMMARY gpurun_out/ab_mintiles.log
