#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of the small cases (profiles/r02_sanitizer_*.log)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  fast=0; [ "$tool" = "racecheck" ] && fast=1
  SAN_FAST=$fast timeout 1500 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.log
done
