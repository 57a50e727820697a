#!/bin/bash
# A/B bench of environment settings: ABS="X=1;Y=2;..." (each run: bench + CTA-0/1 tile trace)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-ab}
: > gpurun_out/${T}.log
IFS=';' read -ra SETS <<< "${ABS:-NONE=1}"
for S in "${SETS[@]}"; do
  echo "=== $S" >> gpurun_out/${T}.log
  env $S timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e $BARGS >> gpurun_out/${T}.log 2>&1
  for C in ${TRACE_CTAS:-0 1}; do
    env $S CTRI_TILE_TRACE=$C timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph $BARGS 2>&1 | grep "tile trace" | head -1 | sed "s/^/cta$C /" >> gpurun_out/${T}.log
  done
done
