#!/bin/bash
# cooperative + PDL launch of the P2P kernel for virtual rows (A) vs cooperative only (B); measured
# no difference (profiles/r2_coop_pdl_ab.txt), so the experiment's CTRI_COOP_NO_PDL code was removed
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-cp}
ng=$(nvidia-smi -L | wc -l)
for cfg in cfg2 cfg4_d1; do
for n in 2 4; do
  [ $n -gt $ng ] && continue
  for v in A B A B; do
    echo "== $cfg N=$n $v" >> gpurun_out/${T}.log
    if [ $v = B ]; then export CTRI_COOP_NO_PDL=1; else unset CTRI_COOP_NO_PDL; fi
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py --config $cfg --gpus $n --steps 50 --warmup 10 \
      --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
  done
done
done
unset CTRI_COOP_NO_PDL
timeout 600 python -m pytest tests/test_multi_gpu.py -q -x -k "2 or 4" > gpurun_out/${T}_mgpu.log 2>&1; echo rc=$? >> gpurun_out/${T}_mgpu.log
python scripts/show_scale.py gpurun_out/${T}.log > gpurun_out/${T}.txt 2>&1
