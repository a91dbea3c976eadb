#!/bin/bash
# ncu --set full of the four config-5 kernels that dominate the cycle (one launch each)
python -m paper_1903_10367_b200.build > /dev/null 2>&1
CMD="python tools/run_cycles.py config5 2"
$CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
for kv in "k3_top2 0" "k3_smooth2r 0" "k3_down_c 0" "k3_up_tile 3"; do
  set -- $kv
  ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
done
