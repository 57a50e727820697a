#!/bin/bash
# cfg2 at N=1: tile variant x virtual partitions -> gpurun_out/sweep_vp.log
mkdir -p gpurun_out
for vp in ${VPS:-1 2 4}; do
  for v in ${VARIANTS:-c16t256s1 c16t512s1 c16t256x3}; do
    echo "== $v vp=$vp" >> gpurun_out/sweep_vp.log
    CTRI_VPARTS=$vp CTRI_TILE_VARIANT=$v timeout 300 python bench.py --steps 300 --warmup 10 \
      --no-cpu-baseline --no-e2e >> gpurun_out/sweep_vp.log 2>&1
  done
done
