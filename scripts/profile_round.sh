#!/bin/bash
# ncu evidence for profiles/: full sets of the hot kernels + a launch list (1 GPU).
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
# cfg2: tile kernel + local reduced/window kernel
$B > gpurun_out/p_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_reduced_local" -s 6 -c 2 \
    -o gpurun_out/prof_cfg2_final $B > gpurun_out/ncu_cfg2.log 2>&1
# launch list of the same run
$B > gpurun_out/p_cfg2b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
    $B > gpurun_out/ncu_launch.log 2>&1
# contiguous axis (index 2)
$B --config cfg4_d2 > gpurun_out/p_d2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 \
    -o gpurun_out/prof_cfg4d2_final $B --config cfg4_d2 > gpurun_out/ncu_d2.log 2>&1
# fused compact derivative (cfg5 at N=1)
$B --config cfg5 > gpurun_out/p_cfg5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 \
    -o gpurun_out/prof_cfg5_final $B --config cfg5 > gpurun_out/ncu_cfg5.log 2>&1
