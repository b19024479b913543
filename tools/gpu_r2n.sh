#!/bin/bash
mkdir -p gpurun_out
python tools/game_levels.py battleship11 cfr 64 2>&1 | sed -n 2,8p
python tools/game_levels.py battleship11 cfr 32 2>&1 | sed -n 2,8p
timeout 900 python tools/ab_flags.py 40 64 0 cfr > gpurun_out/syn_cfr.log 2>&1; cat gpurun_out/syn_cfr.log
timeout 900 python tools/stream_cfg_sweep.py 64 2:0:0 > gpurun_out/sweep_syn.log 2>&1; cat gpurun_out/sweep_syn.log
timeout 900 python -m pytest tests -q -m gpu -x -k "stream or bench_shaped or sharded or parity or variants" > gpurun_out/gpu_stream_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_stream_tests.log
