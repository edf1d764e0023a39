#!/bin/bash
# quick metric capture of one per-layer decode launch (cfg2 step)
mkdir -p gpurun_out
timeout 600 ncu --clock-control none -k regex:decode_kernel -s 8 -c 1 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_ldgsts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_wait_per_warp_active.pct python tools/profile_step.py --steps 1 2>&1 | grep -E "decode_kernel|gpu__|smsp__|l1tex" | head -20
