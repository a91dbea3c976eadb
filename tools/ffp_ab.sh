#!/bin/bash
# A/B of the fused fine pass against the phase-by-phase cycle on config 5 + one ncu capture of k3_ffp4
bash tools/ab.sh config5 "TMG_FFP=0" "TMG_FFP=4"
TMG_FFP=4 python tools/run_cycles.py config5 3 > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
TMG_FFP=4 ncu --set full --clock-control none --import-source on -k regex:k3_ffp4 -s 1 -c 1 -o gpurun_out/prof_ffp4 python tools/run_cycles.py config5 3 > gpurun_out/ncu_ffp4.log 2>&1; echo "ncu rc=$?"
