#!/bin/bash
# Bench every cluster-tile variant on one config (default cfg2) -> gpurun_out/sweep_<cfg>.log
cfg=${1:-cfg2}
steps=${2:-300}
mkdir -p gpurun_out
for v in ${VARIANTS:-c16t512s1 c16t256s1 c16t256x3 c16t512x5 c16t256x6}; do
  echo "== $v" >> gpurun_out/sweep_$cfg.log
  CTRI_TILE_VARIANT=$v timeout 300 python bench.py --config $cfg --steps $steps --warmup 10 \
      --no-cpu-baseline --no-e2e >> gpurun_out/sweep_$cfg.log 2>&1
done
