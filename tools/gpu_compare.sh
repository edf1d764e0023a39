#!/bin/bash
# warp-plan vs split schedules on every decode workload (one line each, key fields)
mkdir -p gpurun_out
show() { python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$1', d['config']['workload'][:5], d['value'], d.get('ms_per_step'), 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'] if d.get('e2e') else None, d['config'].get('schedule'))
"; }
for s in wp split; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-tpot --schedule $s 2>/dev/null | show $s
  timeout 900 python bench.py --workload cfg3 --steps 5 --warmup 3 --schedule $s 2>/dev/null | show $s
  timeout 900 python bench.py --workload cfg4 --steps 5 --warmup 3 --schedule $s 2>/dev/null | show $s
  timeout 600 python bench.py --workload cfg1 --steps 20 --warmup 5 --schedule $s 2>/dev/null | show $s
done
