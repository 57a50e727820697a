#!/bin/bash
# a few ncu metrics of the cfg2 tile kernel: the chain (default) vs the separate-kernel path
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
M="gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_lsu.sum,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_barrier_per_warp_active.pct,smsp__warp_issue_stalled_membar_per_warp_active.pct,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed"
$B > gpurun_out/nm_plain.log 2>&1 && ncu --metrics $M --clock-control none -k regex:k_tile -s 3 -c 1 --csv $B > gpurun_out/nm_vc.csv 2>/dev/null
CTRI_NO_VCHAIN=1 $B > gpurun_out/nm_plain2.log 2>&1 && CTRI_NO_VCHAIN=1 ncu --metrics $M --clock-control none -k regex:k_tile -s 3 -c 1 --csv $B > gpurun_out/nm_old.csv 2>/dev/null
