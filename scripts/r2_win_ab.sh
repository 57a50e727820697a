#!/bin/bash
# window kernel A/B: parity subset, then ncu launch times of the pair kernel vs the per-column one
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-wa}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vchain.py -q -x -k "${PYK:-loopback or window or virtual_rows or acyclic or deriv or detach}" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for shape in "4 256" "2 4096" "4 2048"; do
  for v1 in 0 1; do
    echo "== shape $shape v1=$v1" >> gpurun_out/${T}_ncu.txt
    # (v1 = 1 ran the per-column kernel through a since-removed A/B knob)
    ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_window python scripts/loop_cfg3.py $shape 2>/dev/null | grep '^"' | tail -3 | awk -F'","' '{print $5, $NF}' >> gpurun_out/${T}_ncu.txt
  done
done
unset CTRI_WINDOW_V1
