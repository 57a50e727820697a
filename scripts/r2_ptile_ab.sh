#!/bin/bash
# k_ptile head-PCR A/B (shuffles vs exchange-slot ping-pong; the ping-pong measured 5% slower and was
# removed with its CTRI_PTILE_PCR_SMEM knob) and the column-pair penta window
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-pa}
timeout 900 python -m pytest tests/test_gpu_penta.py -q -x > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
CTRI_PTILE_PCR_SMEM=1 timeout 900 python -m pytest tests/test_gpu_penta.py -q -x -k "on_chip or cfg2_grid or virtual" > gpurun_out/${T}_pytest_smem.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest_smem.log
for i in 1 2 3; do
  timeout 300 python bench.py --penta --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_A$i.log 2>&1
  CTRI_PTILE_PCR_SMEM=1 timeout 300 python bench.py --penta --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_B$i.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_penta_window|k_ptile" -s 6 -c 6 python bench.py --penta --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>/dev/null | grep '^"' > gpurun_out/${T}_ncu.csv
