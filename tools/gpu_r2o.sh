#!/bin/bash
mkdir -p gpurun_out
for v in "" noilp4 "" noilp4; do
  CFR_B200_LIB_VARIANT=$v timeout 900 python tools/stream_cfg_sweep.py 64 2:0:0 2>&1 | head -1 | sed "s/^/[$v] /"
done
