#!/bin/bash
# round-2 evidence on one B200: launch lists (cfg2, penta cfg2 grid, cfg5) and one ncu --set full
# capture of the dominant kernel of cfg2 and of the pentadiagonal solve, summarised to json/txt
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
$B > gpurun_out/r2p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 12 --csv --log-file gpurun_out/r2p_launches_cfg2.csv $B > /dev/null 2>&1
$B --penta > gpurun_out/r2p_plain_penta.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 9 -c 12 --csv --log-file gpurun_out/r2p_launches_penta.csv $B --penta > /dev/null 2>&1
$B --config cfg5 > gpurun_out/r2p_plain_cfg5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 12 --csv --log-file gpurun_out/r2p_launches_cfg5.csv $B --config cfg5 > /dev/null 2>&1
TAG=r2p_ncu_cfg2 KREGEX="k_tile" SKIP=3 bash scripts/ncu_one.sh
TAG=r2p_ncu_penta KREGEX="k_ptile" SKIP=3 bash scripts/ncu_one.sh --penta
TAG=r2p_ncu_cfg5 KREGEX="k_tile" SKIP=3 bash scripts/ncu_one.sh --config cfg5
