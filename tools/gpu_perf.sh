#!/bin/bash
# dev iteration: cfg2 bench (value / single launch / e2e / parity), wp timeline, cfg5 quantize
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-tpot "$@" 2>/dev/null | tail -1 > gpurun_out/bq.json
python -c "import json; d=json.load(open('gpurun_out/bq.json')); print(d['value'], d['roofline']['frac'], 'single', d['single_launch_all_layers_gbs'], 'e2e', d['e2e']['value'], d['clocks'], d.get('parity_sampled_max_rel'))"
timeout 300 python tools/wp_timeline.py 2>&1 | tail -12
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', d['value'], d['unit'], d.get('ms_per_step'), d.get('roofline',{}).get('frac'))"
