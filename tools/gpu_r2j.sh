#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/stream_prof.py 40 > gpurun_out/sprof.log 2>&1; echo "sprof rc=$?"; cat gpurun_out/sprof.log
