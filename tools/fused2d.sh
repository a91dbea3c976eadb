#!/bin/bash
# 2D fused one-launch cycle vs level launches: GPU parity tests, then configs 1, 2, 4 both ways
mkdir -p gpurun_out
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_runner.py -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest.log
for w in config1 config2 config4; do
  for f in "" "--fused-cycle"; do
    timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu --no-ttt $f > gpurun_out/f2d.json 2> gpurun_out/f2d.err || { echo "bench failed $w $f"; tail -3 gpurun_out/f2d.err; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/f2d.json')); print('$w [$f]', round(d['ms_per_step']*1e3,1), 'us', d['gpu_launches'], 'launches', {k: round(v*1e3,1) for k,v in d['kernel_ms'].items()})"
  done
done
