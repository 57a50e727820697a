#!/bin/bash
# one ncu --set full capture of one kernel launch of a bench command, summarised to text:
#   TAG=<name> KREGEX=<kernel regex> SKIP=<launches to skip> bash scripts/ncu_one.sh <bench args...>
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph $*"
$B > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_tile}" -s ${SKIP:-3} -c 1 \
    -o gpurun_out/${TAG} $B > gpurun_out/${TAG}_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/${TAG}.ncu-rep > gpurun_out/${TAG}_sum.json 2>&1
python scripts/ncu_hotspots.py gpurun_out/${TAG}.ncu-rep 14 > gpurun_out/${TAG}_hot.txt 2>&1
rm -f gpurun_out/${TAG}.ncu-rep
