#!/bin/bash
# splits sweep of the per-layer decode bench (+ the batched GPU tests first)
python -m pytest tests/test_gpu_batched.py -q -x 2>&1 | tail -1
for s in ${SPLITS:-9 18 27 36}; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --splits $s 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splits', $s, d['value'], d['ms_per_step'], d['single_launch_all_layers_gbs'])"
done
