#!/bin/bash
# quick metric capture of one reorder/quantize/pack launch (cfg5 prefill)
mkdir -p gpurun_out
timeout 600 ncu --clock-control none -k regex:reorder_quantize -c 1 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,smsp__warps_active.avg.pct_of_peak_sustained_active,smsp__pcsamp_warps_issue_stalled_long_scoreboard.sum,smsp__pcsamp_sample_count.sum,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,sm__warps_active.avg.per_cycle_active python tools/prefill_bench.py 2>&1 | grep -E "reorder|gpu__|smsp__|dram__|launch__|sm__" | head -30
