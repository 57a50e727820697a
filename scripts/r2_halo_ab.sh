#!/bin/bash
# derivative halo rows by TMA from the halo planes (default) vs per-thread loads (CTRI_HALO_GATHER=1,
# an A/B knob removed after this measurement: profiles/r2_halo_tma_ab.txt)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-ha}
timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity.py tests/test_gpu_allgather.py -q -x -k "deriv or compact or stagger or cfg5" > gpurun_out/${T}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_pytest.log
ng=$(nvidia-smi -L | wc -l)
for n in 2 4; do
  [ $n -gt $ng ] && continue
  for v in A B A B; do
    echo "== cfg5 N=$n $v" >> gpurun_out/${T}.log
    if [ $v = B ]; then export CTRI_HALO_GATHER=1; else unset CTRI_HALO_GATHER; fi
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py --config cfg5 --gpus $n --steps 100 --warmup 10 \
      --no-cpu-baseline --no-e2e >> gpurun_out/${T}.log 2>&1
  done
done
unset CTRI_HALO_GATHER
python scripts/show_scale.py gpurun_out/${T}.log > gpurun_out/${T}.txt 2>&1
