#!/bin/bash
# A/B of a decode option flag (bench + timeline), gpu tests first
python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for mode in "" "$@"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill $mode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$mode]', {k:d[k] for k in ['value','ms_per_step','single_launch_all_layers_gbs']})"
  timeout 300 python tools/decode_timeline.py $mode 2>&1 | grep -E "spacing|per-warp tile|final split"
done
