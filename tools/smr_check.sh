#!/bin/bash
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity3d.py -m gpu -x -q > gpurun_out/pytest3d.log 2>&1; echo "pytest3d rc=$?"; tail -3 gpurun_out/pytest3d.log
bash tools/ab.sh config5 TMG_SMR=0 TMG_SMR=1
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print({k: round(v,3) for k,v in d['kernel_ms'].items()})"
