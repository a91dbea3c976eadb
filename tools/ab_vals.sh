#!/bin/bash
# bench config5 for several values of an environment variable: bash tools/ab_vals.sh VAR v1 v2 ... [-- workload]
V=$1; shift
W=config5
for x in "$@"; do
  env $V=$x python bench.py --workload $W --steps 10 --warmup 3 --no-cpu --no-ttt > gpurun_out/ab_${V}_$x.json 2> gpurun_out/ab_${V}_$x.err; echo "$V=$x rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/ab_${V}_$x.json')); print(round(d['ms_per_step'],3), 'ms', 'l2h', d.get('detail',{}).get('l2h_last')); print({k: round(v,3) for k,v in list(d['kernel_ms'].items())[:2]})"
done
