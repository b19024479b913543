#!/bin/bash
for v in "" noilp4; do
  for p in 64 32; do
    CFR_B200_LIB_VARIANT=$v python tools/game_levels.py battleship11 cfr $p 2>&1 | sed -n 2p | sed "s/^/[$v f$p] /"
  done
done
