#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/loop_cfg3.py 4 256 > gpurun_out/c3_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv python scripts/loop_cfg3.py 4 256 > gpurun_out/c3_ncu.csv 2> gpurun_out/c3_ncu.err
ncu --set full --clock-control none -k regex:k_window -s 2 -c 1 -o gpurun_out/c3_window python scripts/loop_cfg3.py 4 256 > gpurun_out/c3_full.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python scripts/loop_cfg3.py 4 512 > gpurun_out/c5like_ncu.csv 2>&1
