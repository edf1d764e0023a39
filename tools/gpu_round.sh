#!/bin/bash
# One GPU session: tests, smoke, full bench (ours + reference arm), every workload, launch list,
# full ncu captures of the decode kernels (warp plan and split) and the quantize kernel.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
timeout 900 python bench.py --workload cfg3 --steps 10 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_cfg3.json
timeout 900 python bench.py --workload cfg3 --cfg3-split head --steps 10 --warmup 3 2>/dev/null | tail -1 >> gpurun_out/bench_cfg3.json
timeout 600 python bench.py --workload cfg1 --steps 30 --warmup 5 2>/dev/null | tail -1 > gpurun_out/bench_cfg1.json
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_cfg5.json
for mp in skewed all_int2 all_fp16; do timeout 900 python bench.py --workload cfg4 --cfg4-map $mp --steps 10 --warmup 3 2>/dev/null | tail -1; done > gpurun_out/bench_cfg4.jsonl
timeout 900 python bench.py --chains 1 --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-tpot 2>/dev/null | tail -1 > gpurun_out/bench_lockstep.json
timeout 900 python bench.py --chains 1 --schedule split --steps 10 --warmup 3 --no-cpu-baseline --no-prefill --no-tpot 2>/dev/null | tail -1 > gpurun_out/bench_split.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 --prefill > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:decode_kernel -s 64 -c 1 -o gpurun_out/decode_chain_prof -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_decode_chain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:decode_wp_kernel -s 8 -c 1 -o gpurun_out/decode_prof -f python tools/profile_step.py --steps 1 --chains 1 > gpurun_out/ncu_decode.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:decode_kernel -s 8 -c 1 -o gpurun_out/decode_split_prof -f python tools/profile_step.py --steps 1 --chains 1 --schedule split > gpurun_out/ncu_decode_split.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:reorder_quantize -c 1 -o gpurun_out/quant_prof -f python tools/profile_step.py --steps 1 --layers 1 --prefill > gpurun_out/ncu_quant.log 2>&1
tail -n 1 gpurun_out/ncu_decode.log; tail -n 1 gpurun_out/ncu_quant.log
