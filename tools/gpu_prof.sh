#!/bin/bash
# ncu capture of the decode kernel (per-layer launch) and launch list for one step
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 40 -c 1 -o gpurun_out/decode_prof -f python tools/profile_step.py --steps 2 > gpurun_out/ncu_decode.log 2>&1
tail -2 gpurun_out/ncu_decode.log
