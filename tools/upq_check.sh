#!/bin/bash
# k3_up_tma: parity vs k3_up_tile, A/B on config 5, one ncu capture
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity3d.py -m gpu -x -q -k "stream or fixture or level3" > gpurun_out/pytest_upq.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_upq.log
bash tools/ab.sh config5 "TMG_UPQ=0" "TMG_UPQ=1"
python tools/run_cycles.py config5 2 > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k3_up_tma -s 0 -c 1 -o gpurun_out/prof_k3_up_tma python tools/run_cycles.py config5 2 > gpurun_out/ncu_upq.log 2>&1; echo "ncu rc=$?"
