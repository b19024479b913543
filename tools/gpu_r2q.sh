#!/bin/bash
# full GPU suite, smoke, default bench on the current tree
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])
for e in d['per_game']: print(e['game'], e['variant'], e['dtype'], e['it_per_s'], e.get('oracle',{}).get('it_per_s'), e.get('paper_context',{}).get('ratio'))
for e in d['synthetic_variants']: print(e)
"
