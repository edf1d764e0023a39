#!/bin/bash
# quick GPU iteration: gpu tests + bench without cpu baseline
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>&1 | tail -2
