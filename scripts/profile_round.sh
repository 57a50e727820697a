#!/bin/bash
# ncu evidence for profiles/: full sets of the hot kernels + a launch list (1 GPU).  Every
# ncu command runs only after the same bench command exited 0 without ncu.
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
# cfg2: tile kernel + local reduced system + window pass
$B > gpurun_out/p_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_reduced_local|k_window" -s 9 -c 3 \
    -o gpurun_out/prof_cfg2_final $B > gpurun_out/ncu_cfg2.log 2>&1
# launch list of the same run
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
    $B > gpurun_out/ncu_launch.log 2>&1
# contiguous axis (index 2): zero-padding TMA tile kernel
$B --config cfg4_d2 > gpurun_out/p_d2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 \
    -o gpurun_out/prof_cfg4d2_final $B --config cfg4_d2 > gpurun_out/ncu_d2.log 2>&1
# fused compact derivative (cfg5 at N=1)
$B --config cfg5 > gpurun_out/p_cfg5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 \
    -o gpurun_out/prof_cfg5_final $B --config cfg5 > gpurun_out/ncu_cfg5.log 2>&1
# weak-scaling slab (cfg3 at N=1)
$B --config cfg3 > gpurun_out/p_cfg3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 \
    -o gpurun_out/prof_cfg3_final $B --config cfg3 > gpurun_out/ncu_cfg3.log 2>&1
# pentadiagonal column-serial local solve (N3)
$B --penta > gpurun_out/p_penta.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_penta_local -s 3 -c 1 \
    -o gpurun_out/prof_penta_final $B --penta > gpurun_out/ncu_penta.log 2>&1
# summaries (the .ncu-rep files stay on the box: gpurun copies back <= 64 MiB)
for r in cfg2 cfg4d2 cfg5 cfg3 penta; do
  [ -f gpurun_out/prof_${r}_final.ncu-rep ] && \
    python scripts/ncu_summary.py gpurun_out/prof_${r}_final.ncu-rep > gpurun_out/sum_${r}.json 2>&1
done
python scripts/ncu_hotspots.py gpurun_out/prof_cfg4d2_final.ncu-rep > gpurun_out/hot_cfg4d2.txt 2>&1
rm -f gpurun_out/prof_cfg3_final.ncu-rep gpurun_out/prof_penta_final.ncu-rep gpurun_out/prof_cfg5_final.ncu-rep \
      gpurun_out/prof_cfg2_final.ncu-rep
