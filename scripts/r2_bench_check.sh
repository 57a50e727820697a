#!/bin/bash
# the bench after timing without phase events: N=1 (cfg2, cfg5, penta) and N=2/4 (cfg2, cfg3, cfg5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-bc}
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_default.log 2>&1
echo "== cfg2 N=1" >> gpurun_out/${T}.log; timeout 300 python bench.py --config cfg2 --steps 50 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
echo "== cfg5 N=1" >> gpurun_out/${T}.log; timeout 300 python bench.py --config cfg5 --steps 50 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
echo "== cfg3 N=1" >> gpurun_out/${T}.log; timeout 300 python bench.py --config cfg3 --steps 50 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
echo "== cfg4_d2 N=1" >> gpurun_out/${T}.log; timeout 300 python bench.py --config cfg4_d2 --steps 50 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
echo "== penta N=1" >> gpurun_out/${T}.log; timeout 300 python bench.py --config cfg2 --penta --steps 50 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
ng=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  [ $n -gt $ng ] && continue
  for spec in "cfg2" "cfg3" "cfg4_d1" "cfg4_d2" "cfg5" "cfg2 --penta"; do
    echo "== $spec N=$n" >> gpurun_out/${T}.log
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py --config $spec --gpus $n --steps 50 --warmup 10 \
      --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
  done
done
python scripts/show_scale.py gpurun_out/${T}.log > gpurun_out/${T}.txt 2>&1
