#!/bin/bash
# per-tile phase trace of k_ptile (pentadiagonal on chip) next to k_tile's, plus a parity subset
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-pt}
if [ -n "$PYK" ]; then
  timeout 900 python -m pytest tests/ -m gpu -x -q -k "$PYK" > gpurun_out/${T}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
fi
for cta in 0 101 202; do
  echo "== penta cta $cta" >> gpurun_out/${T}_trace.log
  CTRI_TILE_TRACE=$cta timeout 120 python bench.py --penta --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>&1 | grep "trace" | tail -2 >> gpurun_out/${T}_trace.log
  echo "== k_tile (three-kernel path) cta $cta" >> gpurun_out/${T}_trace.log
  CTRI_NO_VCHAIN=1 CTRI_TILE_TRACE=$cta timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>&1 | grep "trace" | tail -2 >> gpurun_out/${T}_trace.log
done
timeout 300 python bench.py --penta --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_penta.log 2>&1
