#!/bin/bash
# compute-sanitizer on a few cycles of a workload: bash tools/sanitize.sh WORKLOAD [ENV...]
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || exit 1
w=$1; shift
env "$@" timeout 600 compute-sanitizer --tool memcheck python tools/ffp_probe.py $w 2 > gpurun_out/sanitize.log 2>&1; echo "rc=$?"
grep -v "^=========     " gpurun_out/sanitize.log | head -40
