#!/bin/bash
# end-of-round-2 scaling on one box: every BASELINE config at N = 1, 2, 4, the pentadiagonal
# cfg2 grid (default: 1024-row partitions as virtual rows; and CTRI_VPARTS=1 at N = 4), the
# multi-GPU parity tests first -> gpurun_out/${T}.log / .txt
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2f}
ng=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multi_gpu.py -q -x > gpurun_out/${T}_mgpu_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_mgpu_pytest.log
run() {  # name, N, env, args...
  local name=$1 n=$2 env=$3; shift 3
  echo "== $name N=$n" >> gpurun_out/${T}.log
  if [ $n -eq 1 ]; then
    env $env timeout 300 python bench.py "$@" --steps ${STEPS:-100} --warmup 10 --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
  else
    env $env timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py "$@" --gpus $n --steps ${STEPS:-100} --warmup 10 \
      --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
  fi
}
for cfg in cfg2 cfg3 cfg4_d1 cfg4_d2 cfg5; do
  for n in 1 2 4; do [ $n -le $ng ] && run $cfg $n "X=1" --config $cfg; done
done
for n in 1 2 4; do [ $n -le $ng ] && run "cfg2-penta" $n "X=1" --config cfg2 --penta; done
[ 4 -le $ng ] && run "cfg2-penta-vp1" 4 "CTRI_VPARTS=1" --config cfg2 --penta
python scripts/show_scale.py gpurun_out/${T}.log > gpurun_out/${T}.txt 2>&1
