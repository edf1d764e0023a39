#!/bin/bash
# FP16-region path A/B: cfg4 2-layer sweep maps under both schedules for each library variant.
# usage: bash tools/gpu_fp16.sh name1 name2 ... (build/variants/<name>.so; "main" = in-tree lib)
for n in "$@"; do
  lib=build/variants/$n.so; [ "$n" = "main" ] && lib=paper_2503_23294_b200/_lib/libckv.so
  for sch in split wp; do
    echo "== $n $sch"
    CKV_LIB_PATH=$PWD/$lib CKV_SCHEDULE=$sch timeout 600 python tools/cfg4_bench.py all_fp16 skewed 2>&1 | tail -2
  done
done
