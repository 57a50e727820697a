#!/bin/bash
# end-of-round check on one B200: the whole GPU suite, smoke(), the default bench (driver
# command) and the reference arm, then the ncu evidence (launch lists + one --set full capture
# per dominant kernel: cfg2 chain, pentadiagonal k_ptile, cfg5 fused stencil)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fin_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/fin_smoke.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_bench.log 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 3 --warmup 3 > gpurun_out/fin_ref.log 2>&1
bash scripts/r2_profile.sh
