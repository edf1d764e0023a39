#!/bin/bash
# iteration: gpu tests, bench (no cpu baseline / prefill), ncu of one decode launch
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-prefill 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','tokens_per_s','single_launch_all_layers_gbs']}, d['roofline']['frac'], d['e2e']['value'], d['config']['splits'], d['clocks'])"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:decode_kernel -s 8 -c 1 -o gpurun_out/decode_prof -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_decode.log 2>&1
tail -n 1 gpurun_out/ncu_decode.log
