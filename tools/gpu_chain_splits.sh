#!/bin/bash
# splits sweep of the chained default step (8 micro-batch chains)
for rep in 1 2; do for s in ${SPLITS:-9 10 11 12 19 20}; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-prefill --no-tpot --no-sustained --splits $s 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('splits $s', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
