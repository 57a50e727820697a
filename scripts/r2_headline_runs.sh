#!/bin/bash
# the driver's N=1 command, five times on one box (headline spread)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-hl}
for i in 1 2 3 4 5; do
  timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_$i.log 2>&1
done
nvidia-smi --query-gpu=name,serial,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt 2>&1
