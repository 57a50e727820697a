#!/bin/bash
# Reduced-system variants (pairwise P2P schedule / P2P all-gather / NCCL rounds) at N = 2, 4.
mkdir -p gpurun_out
ng=$(nvidia-smi -L | wc -l)
for cfg in ${CFGS:-cfg2 cfg3}; do
  for n in 2 4; do
    [ $n -gt $ng ] && continue
    for red in ${REDS:-fused pcr allgather nccl}; do
      echo "== $cfg N=$n $red" >> gpurun_out/reduced.log
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29710 + n)) bench.py --config $cfg --gpus $n --steps 300 --warmup 10 \
        --reduced $red --no-cpu-baseline --no-e2e >> gpurun_out/reduced.log 2>&1
    done
  done
done
