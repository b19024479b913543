#!/bin/bash
# early row release with a live-row buffer: parity tests first, then A/B on the synthetic
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -k "stream or fullsize_sampled or battleship or goofspiel6 or bench_shaped or variants" > gpurun_out/gpu_stream_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_stream_tests.log
timeout 900 python tools/ab_env.py 64 0 - CFR_STREAM_LATE_RELEASE=1 > gpurun_out/ab_early64.log 2>&1; grep SUMMARY gpurun_out/ab_early64.log
timeout 900 python tools/ab_env.py 32 0 - CFR_STREAM_LATE_RELEASE=1 > gpurun_out/ab_early32.log 2>&1; grep SUMMARY gpurun_out/ab_early32.log
AB_VARIANT=cfr timeout 900 python tools/ab_env.py 64 0 - CFR_STREAM_LATE_RELEASE=1 > gpurun_out/ab_early64v.log 2>&1; grep SUMMARY gpurun_out/ab_early64v.log
