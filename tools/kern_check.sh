#!/bin/bash
# build, 3D GPU parity, A/B of env knobs on config 5: bash tools/kern_check.sh "ENV1" "ENV2" ...
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity3d.py -m gpu -x -q > gpurun_out/pytest3d.log 2>&1; echo "pytest3d rc=$?"; tail -3 gpurun_out/pytest3d.log
bash tools/ab.sh config5 "$@"
