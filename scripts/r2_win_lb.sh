#!/bin/bash
# (measured slightly slower than the default register budget -- cfg3 slab 17.1-17.7 vs 16.3-17.4 us,
# penta 199 vs 185 us -- and not kept)
# window passes with __launch_bounds__(256, 4) (4 CTAs per SM): ncu launch times (cold) for the
# cfg3 slab, cfg2 N=2 / N=4 shapes (loopback) and the pentadiagonal grid; parity subset
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-wl}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_penta.py -q -x -k "loopback or window or virtual or on_chip or cfg2_grid or layouts" > gpurun_out/${T}_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_pytest.log
for shape in "4 256" "2 4096" "4 2048"; do
  echo "== shape $shape" >> gpurun_out/${T}_ncu.txt
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_window python scripts/loop_cfg3.py $shape 2>/dev/null | grep '^"' | tail -3 | awk -F'","' '{print $5, $NF}' >> gpurun_out/${T}_ncu.txt
done
echo "== penta" >> gpurun_out/${T}_ncu.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_penta_window -s 2 -c 3 python bench.py --penta --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>/dev/null | grep '^"' | awk -F'","' '{print $5, $NF}' >> gpurun_out/${T}_ncu.txt
