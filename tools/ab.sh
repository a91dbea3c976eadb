#!/bin/bash
# A/B of environment variants on one workload: bash tools/ab.sh WORKLOAD "ENV1" "ENV2" ...
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
w=$1; shift
for v in "$@"; do
  env $v python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-ttt > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$v failed"; tail -3 gpurun_out/ab.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; print('$v', round(d['ms_per_step'],3), 'ms', {x: round(y,3) for x,y in k.items() if y > 0.2})"
done
