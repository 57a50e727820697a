#!/bin/bash
# per-tile trace of the chain vs the three-kernel k_tile at early, middle and late tiles
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-vl}
for off in 0 100 160; do
  for cta in 0 101; do
    echo "== chain cta $cta off $off" >> gpurun_out/${T}_trace.log
    CTRI_TILE_TRACE_OFF=$off CTRI_TILE_TRACE=$cta timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>&1 | grep "trace" | tail -1 >> gpurun_out/${T}_trace.log
    echo "== three-kernel cta $cta off $off" >> gpurun_out/${T}_trace.log
    CTRI_NO_VCHAIN=1 CTRI_TILE_TRACE_OFF=$off CTRI_TILE_TRACE=$cta timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>&1 | grep "trace" | tail -1 >> gpurun_out/${T}_trace.log
  done
done
