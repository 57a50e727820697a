#!/bin/bash
# round-2 scaling: every BASELINE config at N = 1, 2, 4 (as many GPUs as the box has), plus the
# pentadiagonal cfg2 grid; per-round comm times in the JSON lines -> gpurun_out/r2_scale.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ng=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/r2_topo.txt 2>&1
for spec in ${SPECS:-"cfg2" "cfg3" "cfg4_d1" "cfg4_d2" "cfg5" "cfg2 --penta"}; do
  for n in 1 2 4 8; do
    [ $n -gt $ng ] && continue
    echo "== $spec N=$n" >> gpurun_out/r2_scale.log
    if [ $n -eq 1 ]; then
      timeout 300 python bench.py --config $spec --steps 300 --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/r2_scale.log 2>&1
    else
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29700 + n)) bench.py --config $spec --gpus $n --steps 300 --warmup 10 \
        --no-cpu-baseline --no-e2e >> gpurun_out/r2_scale.log 2>&1
    fi
  done
done
python scripts/show_scale.py gpurun_out/r2_scale.log > gpurun_out/r2_scale.txt 2>&1
