#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python tools/sub_ab.py goofspiel6 battleship4 battleship6 > gpurun_out/sub_ab7.log 2>&1; cat gpurun_out/sub_ab7.log
timeout 900 python tools/sub_cut_sweep.py goofspiel6 battleship6 > gpurun_out/sub_cut3.log 2>&1; cat gpurun_out/sub_cut3.log
