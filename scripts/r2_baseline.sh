#!/bin/bash
# round-2 baseline: gpu tests and bench (compute-sanitizer is closed on this pool)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -q | grep -A3 -i "Product Name" | head -8 > gpurun_out/r2b_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 300 python bench.py --steps 200 --warmup 10 > gpurun_out/r2b_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2b_bench.log
