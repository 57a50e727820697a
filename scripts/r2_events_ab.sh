#!/bin/bash
# does the plan's per-phase event recording (CTRI_FLAG_TIMING, event nodes between the kernels
# of a captured solve) cost time?  A = with (the bench default), B = --no-phase-events
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-ev}
ng=$(nvidia-smi -L | wc -l)
run() {  # name n args...
  local name=$1 n=$2; shift 2
  for v in A B A B; do
    echo "== $name N=$n $v" >> gpurun_out/${T}.log
    extra=""; [ $v = B ] && extra="--no-phase-events"
    if [ $n -eq 1 ]; then
      timeout 300 python bench.py "$@" $extra --steps 50 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'])" >> gpurun_out/${T}.log
    else
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29700 + n)) bench.py "$@" $extra --gpus $n --steps 50 --warmup 10 \
        --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'])" >> gpurun_out/${T}.log
    fi
  done
}
run "penta" 1 --config cfg2 --penta
run "cfg4_d2" 1 --config cfg4_d2
for n in 2 4; do
  [ $n -gt $ng ] && continue
  run cfg2 $n --config cfg2
  run cfg5 $n --config cfg5
  run cfg3 $n --config cfg3
done
