#!/bin/bash
# A/B of an environment switch on the config-5 bench: bash tools/ab_env.sh VAR [workload]
V=$1; W=${2:-config5}
for x in 1 0; do
  env $V=$x python bench.py --workload $W --steps 10 --warmup 3 --no-cpu --no-ttt > gpurun_out/ab_${V}_$x.json 2> gpurun_out/ab_${V}_$x.err; echo "$V=$x rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/ab_${V}_$x.json')); print(round(d['ms_per_step'],3), 'ms'); print({k: round(v,3) for k,v in d['kernel_ms'].items()})"
done
