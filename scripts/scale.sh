#!/bin/bash
# Strong (cfg2) and weak (cfg3) scaling at N = 1, 2, 4, 8 (as many GPUs as the box has).
mkdir -p gpurun_out
ng=$(nvidia-smi -L | wc -l)
for cfg in ${CFGS:-cfg2 cfg3}; do
  for n in 1 2 4 8; do
    [ $n -gt $ng ] && continue
    echo "== $cfg N=$n" >> gpurun_out/scale.log
    if [ $n -eq 1 ]; then
      timeout 300 python bench.py --config $cfg --steps 300 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/scale.log 2>&1
    else
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29700 + n)) bench.py --config $cfg --gpus $n --steps 300 --warmup 10 \
        --no-cpu-baseline --no-e2e >> gpurun_out/scale.log 2>&1
    fi
  done
done
