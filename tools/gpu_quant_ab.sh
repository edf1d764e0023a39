#!/bin/bash
# quantize kernel A/B: DRAM bytes, instructions and duration of one cfg5 launch (ncu) and the
# prefill timing (no profiler) per library variant. usage: bash tools/gpu_quant_ab.sh name ...
for n in "$@"; do
  lib=build/variants/$n.so; [ "$n" = "main" ] && lib=paper_2503_23294_b200/_lib/libckv.so
  echo "== $n"
  CKV_LIB_PATH=$PWD/$lib timeout 600 python tools/prefill_bench.py 2>&1 | tail -1 | cut -c1-200
  CKV_LIB_PATH=$PWD/$lib timeout 600 ncu --clock-control none -k regex:reorder_quantize -c 1 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread python tools/prefill_bench.py 2>&1 | grep -E "gpu__|smsp__|dram__|launch__"
done
