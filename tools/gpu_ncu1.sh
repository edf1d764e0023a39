#!/bin/bash
# one full ncu capture of a per-layer decode launch (steady state) + summary
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:decode_kernel -s 8 -c 1 -o gpurun_out/${1:-decode_prof} -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_decode.log 2>&1
tail -n 2 gpurun_out/ncu_decode.log
