#!/bin/bash
# dev iteration: gpu tests, short cfg2 bench (value / single launch), wp timeline
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-tpot "$@" 2>/dev/null | tail -1 > gpurun_out/bq.json
python -c "import json; d=json.load(open('gpurun_out/bq.json')); print(d['value'], d['roofline']['frac'], 'single', d['single_launch_all_layers_gbs'], 'e2e', d['e2e']['value'], d['clocks'], d.get('parity_sampled_max_rel'))"
timeout 300 python tools/wp_timeline.py 2>&1 | tail -14
