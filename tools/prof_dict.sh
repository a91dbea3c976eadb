#!/bin/bash
# ncu --set full of the dictionary-variant smr / up kernels at config 5 (one launch each)
python -m paper_1903_10367_b200.build > /dev/null 2>&1
CMD="python tools/run_cycles.py config5 2"
$CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
for k in ${KERNELS:-k3_smr k3_up_dict}; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-0} -c 1 -o gpurun_out/prof_dict_$k $CMD > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
  python tools/ncu_brief.py gpurun_out/prof_dict_$k.ncu-rep
done
