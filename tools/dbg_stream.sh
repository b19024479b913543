for d in 0 16 32 48 20; do CFR_STREAM_DEBUG=$d timeout 600 python tools/stream_prof.py 40 2>&1 | tail -1 ; echo " debug=$d"; done
