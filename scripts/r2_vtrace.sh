#!/bin/bash
# per-tile phase trace of the virtual-partition chain (k_tile LAYOUT 4) next to the three-kernel
# path's k_tile (LAYOUT 0), same CTAs; then the penta bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-vt}
for cta in 0 101 202; do
  echo "== chain cta $cta" >> gpurun_out/${T}_trace.log
  CTRI_TILE_TRACE=$cta timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>&1 | grep "trace" | tail -2 >> gpurun_out/${T}_trace.log
  echo "== three-kernel k_tile cta $cta" >> gpurun_out/${T}_trace.log
  CTRI_NO_VCHAIN=1 CTRI_TILE_TRACE=$cta timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>&1 | grep "trace" | tail -2 >> gpurun_out/${T}_trace.log
done
for i in 1 2; do
timeout 300 python bench.py --penta --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_penta$i.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench$i.log 2>&1
done
