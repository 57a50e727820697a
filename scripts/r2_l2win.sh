#!/bin/bash
# A/B of the L2-resident window rows (CTRI_L2_WINDOW_MB=0 disables) on the multi-GPU configs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for spec in cfg5 cfg3 cfg4_d1; do
  for n in 2 4; do
    for cap in 0 256; do
      echo "== $spec N=$n l2cap=$cap" >> gpurun_out/r2_l2win.log
      CTRI_L2_WINDOW_MB=$cap timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29700 + n)) bench.py --config $spec --gpus $n --steps 300 --warmup 10 \
        --no-cpu-baseline --no-e2e >> gpurun_out/r2_l2win.log 2>&1
    done
  done
done
python scripts/show_scale.py gpurun_out/r2_l2win.log > gpurun_out/r2_l2win.txt 2>&1
