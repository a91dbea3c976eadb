#!/bin/bash
# weight dictionaries: parity tests, storage of config 5, A/B against the dense streams
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity3d.py -m gpu -x -q -k "dictionary or stream_equals or fixture" > gpurun_out/pytest_dict.log 2>&1; echo "pytest dict rc=$?"; tail -5 gpurun_out/pytest_dict.log
bash tools/ab.sh config5 TMG_PDICT=0 TMG_PDICT_SMR=0 TMG_PDICT=1
