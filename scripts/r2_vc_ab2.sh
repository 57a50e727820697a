#!/bin/bash
# A/B inside one call: default chain vs CTRI_VC_DBG=$BITS, plus the three-kernel path
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-vb}
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_A$i.log 2>&1
  CTRI_VC_DBG=$BITS timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_B$i.log 2>&1
done
CTRI_NO_VCHAIN=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_old.log 2>&1
