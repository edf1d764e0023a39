#!/bin/bash
# A/B of decode variants (build/variants/<name>.so): per-layer graph step + single launch.
# usage: bash tools/ab.sh name1 name2 ... [-- extra bench args]
mkdir -p gpurun_out
names=(); extra=()
while [ $# -gt 0 ]; do if [ "$1" = "--" ]; then shift; extra=("$@"); break; fi; names+=("$1"); shift; done
for n in "${names[@]}"; do
  lib=build/variants/$n.so; [ "$n" = "main" ] && lib=paper_2503_23294_b200/_lib/libckv.so
  CKV_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-sustained "${extra[@]}" 2>gpurun_out/ab_$n.err | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$n', {k:d.get(k) for k in ['value','ms_per_step','single_launch_all_layers_gbs','eager_launches_gbs']}, 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'], 'splits', d['config']['splits'], d['config'].get('schedule'), d['clocks']['sm_mhz'], d['clocks']['reasons'])
except Exception as e: print('$n FAILED', e)
"
done
