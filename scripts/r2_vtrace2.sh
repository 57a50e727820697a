#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-vt2}
for cta in 0 101 202 283; do
  echo "== chain cta $cta off 100" >> gpurun_out/${T}_trace.log
  CTRI_TILE_TRACE_OFF=100 CTRI_TILE_TRACE=$cta timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>&1 | grep "trace" | tail -2 >> gpurun_out/${T}_trace.log
done
