#!/bin/bash
# dev iteration: gpu tests, per-layer bench, timeline summary
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','tokens_per_s','single_launch_all_layers_gbs']}, d['roofline']['frac'], d['e2e']['value'], d['config']['splits'], d['clocks'])"
timeout 300 python tools/decode_timeline.py 2>&1 | tail -12
