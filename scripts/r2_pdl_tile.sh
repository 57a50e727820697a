#!/bin/bash
# (measured no difference: cfg5 N=2 0.506, N=4 0.349 ms; the change was not kept)
# the fused derivative's tile kernel launched programmatically after the halo kernel:
# multi-GPU parity and cfg5 at N = 2, 4 (compare profiles/r2_scale_end_noevents.txt: 0.505 / 0.350)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-pt}
timeout 1200 python -m pytest tests/test_multi_gpu.py -q -x -k "2 or 4" > gpurun_out/${T}_mgpu.log 2>&1; echo rc=$? >> gpurun_out/${T}_mgpu.log
for n in 2 4; do
  for i in 1 2; do
    echo "== cfg5 N=$n" >> gpurun_out/${T}.log
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py --config cfg5 --gpus $n --steps 50 --warmup 10 \
      --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
  done
done
python scripts/show_scale.py gpurun_out/${T}.log > gpurun_out/${T}.txt 2>&1
