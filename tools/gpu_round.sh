#!/bin/bash
# One GPU session: tests, bench, launch list, full ncu capture of the decode and quantize kernels.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 --prefill > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 40 -c 2 -o gpurun_out/decode_prof -f python tools/profile_step.py --steps 2 > gpurun_out/ncu_decode.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reorder_quantize -c 1 -o gpurun_out/quant_prof -f python tools/profile_step.py --steps 1 --layers 1 --prefill > gpurun_out/ncu_quant.log 2>&1
tail -3 gpurun_out/ncu_decode.log gpurun_out/ncu_quant.log
ls -la gpurun_out
