for d in 0 4 8 12; do CFR_STREAM_DEBUG=$d CFR_B200_LIB_VARIANT=sprof timeout 600 python tools/stream_prof.py 40 2>&1 | tail -9 | tr '\n' ' ' ; echo " debug=$d"; done
timeout 900 python tools/stream_sweep.py 40 240,2 240,2,4 240,2,8 240,2,12 2>&1 | cut -c1-120
