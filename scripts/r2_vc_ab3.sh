#!/bin/bash
# chain check: parity subset, trace, bench alternating with the three-kernel path
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-vc3}
timeout 900 python -m pytest tests/test_gpu_vchain.py tests/test_gpu_parity.py -q -x -k "${PYK:-vchain or two_level or cfg2_full or virtual}" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for cta in 0 202; do
  echo "== chain cta $cta off 100" >> gpurun_out/${T}_trace.log
  CTRI_TILE_TRACE_OFF=100 CTRI_TILE_TRACE=$cta timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>&1 | grep "trace" | tail -2 >> gpurun_out/${T}_trace.log
done
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench$i.log 2>&1
  CTRI_NO_VCHAIN=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_old$i.log 2>&1
done
