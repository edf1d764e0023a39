#!/bin/bash
# quick metric capture of one reorder/quantize/pack launch (cfg5 prefill)
mkdir -p gpurun_out
timeout 600 ncu --clock-control none -k regex:reorder_quantize -c 1 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,smsp__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.per_cycle_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_shared_ld.sum python tools/prefill_bench.py 2>&1 | grep -E "reorder|gpu__|smsp__|dram__|launch__|sm__|l1tex" | head -30
