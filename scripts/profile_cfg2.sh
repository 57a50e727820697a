mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
$B > gpurun_out/p_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_reduced_local|k_window" -s 9 -c 3 \
    -o gpurun_out/prof_cfg2_final $B > gpurun_out/ncu_cfg2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
    $B > gpurun_out/ncu_launch.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_cfg2_final.ncu-rep > gpurun_out/sum_cfg2.json 2>&1
rm -f gpurun_out/prof_cfg2_final.ncu-rep
