#!/bin/bash
# round-2 baseline: gpu tests, bench, compute-sanitizer on the small cases
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
nvidia-smi -q | grep -A3 -i "GPC\|Product Name" | head -20 > gpurun_out/r2b_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 300 python bench.py --steps 200 --warmup 10 > gpurun_out/r2b_bench.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/r2b_san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r2b_san_$tool.log
done
