#!/bin/bash
# A/B of compile-time variants on one box:  bash tools/ab_flags.sh config5 "" "-DCYC_MINB=2" ...
# (each argument after the workload is a TMG_NVCC_FLAGS value; prints cycle and per-kernel ms)
mkdir -p gpurun_out
W=$1; shift
for rep in 1 2; do
for f in "$@"; do
  TMG_NVCC_FLAGS="$f" python -m paper_1903_10367_b200.build --force > gpurun_out/build.log 2>&1 || { echo "build failed: $f"; tail -5 gpurun_out/build.log; continue; }
  timeout 180 python bench.py --workload $W --steps 30 --warmup 3 --no-cpu --no-ttt > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "bench failed: $f"; tail -3 gpurun_out/ab.err; continue; }
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms']; print('[%s]' % '$f', round(d['ms_per_step'],3), 'ms |', ' '.join('%s %.3f' % (n.replace('k3_',''), v) for n, v in k.items() if v > 0.1))"
done
done
python -m paper_1903_10367_b200.build --force > /dev/null 2>&1
