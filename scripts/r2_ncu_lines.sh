#!/bin/bash
# per-CUDA-source-line instruction counts of the cfg2 tile kernel (the chain)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
$B > gpurun_out/nl_plain.log 2>&1 && ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on -k regex:k_tile -s 3 -c 1 -o gpurun_out/nl_vc $B > gpurun_out/nl_ncu.log 2>&1
