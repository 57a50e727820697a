#!/bin/bash
# E4: 2^n vs 2^n - 1 GPUs, solve index 1, weak scaling (256 x 2048 x 256 per GPU):
# p = 1, 2, 3, 4 on one box (p = 3: detach / reattach of the reduced system)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-e4}
ng=$(nvidia-smi -L | wc -l)
for n in 1 2 3 4; do
  [ $n -gt $ng ] && continue
  d="256,$((2048 * n)),256"
  echo "== index1 weak N=$n dims $d" >> gpurun_out/${T}.log
  if [ $n -eq 1 ]; then
    timeout 300 python bench.py --dims $d --sd 1 --steps 50 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py --dims $d --sd 1 --gpus $n --steps 50 --warmup 10 \
      --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
  fi
done
python scripts/show_scale.py gpurun_out/${T}.log > gpurun_out/${T}.txt 2>&1
