#!/bin/bash
# (the persistent form measured slower -- cfg3 slab 19.9 vs 16.8 us, cfg2 N=2 67 vs 56, N=4 35 vs 29 --
# and was not kept; CTRI_WINDOW_WAVES selected the wave-launched kernel for this A/B only)
# persistent window pass (default) vs the wave-launched one (CTRI_WINDOW_WAVES=1): parity subset,
# ncu launch times (cold) on the cfg3 slab and the cfg2 N=2 / N=4 shapes (loopback)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-wpp}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -q -x -k "loopback or window or virtual or multi_partition or acyclic or detach or deriv or cfg5" > gpurun_out/${T}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_pytest.log
for shape in "4 256" "2 4096" "4 2048"; do
  for v in 0 1; do
    echo "== shape $shape waves=$v" >> gpurun_out/${T}_ncu.txt
    if [ $v = 1 ]; then export CTRI_WINDOW_WAVES=1; else unset CTRI_WINDOW_WAVES; fi
    ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_window python scripts/loop_cfg3.py $shape 2>/dev/null | grep '^"' | tail -3 | awk -F'","' '{print $5, $NF}' >> gpurun_out/${T}_ncu.txt
  done
done
unset CTRI_WINDOW_WAVES
