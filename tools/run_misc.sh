timeout 900 python tools/stream_sweep.py 40 240,2 2>&1 | cut -c1-150
timeout 900 python bench.py --precision 32 --no-cpu --no-games --e2e-steps 5 --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('f32', d['value'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'])"
bash tools/ncu_fwd.sh
