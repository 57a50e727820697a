#!/bin/bash
# quick round-2 iteration: a parity subset, the bench, and the per-tile trace of CTA 0
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-q}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "${PYK:-shapes or bands or loopback_partitions or cfg2}" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench.log 2>&1
CTRI_TILE_TRACE=1 timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>&1 | grep "tile trace" | head -3 >> gpurun_out/${T}_bench.log
if [ -n "$AB" ]; then  # A/B: the same bench with an extra environment setting
  env $AB timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/${T}_benchB.log 2>&1
fi
