#!/bin/bash
# build, 3D parity, quick 3D benches (no CPU leg)
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity3d.py -m gpu -x -q > gpurun_out/pytest3d.log 2>&1; echo "pytest3d rc=$?"; tail -3 gpurun_out/pytest3d.log
for w in ${@:-config3 config5}; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-ttt > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'GDoF/s frac', round(d['roofline']['cycle_frac'],3)); print({k: round(v,3) for k,v in d['kernel_ms'].items()})"
done
