#!/bin/bash
# ncu --set full of the three finest-level kernels of the config-5 cycle (one launch each)
python -m paper_1903_10367_b200.build > /dev/null 2>&1
CMD="python tools/run_cycles.py config5 3"
$CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
for kv in "k3_smr 1" "k3_up_dict 1" "k3_top4 1"; do
  set -- $kv
  ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -f -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
done
