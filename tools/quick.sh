#!/bin/bash
# build, GPU tests (optionally a subset), quick benches without the CPU leg:
#   bash tools/quick.sh "<pytest args>" config5 config3 ...
mkdir -p gpurun_out
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
T=${1:-tests}
timeout 1500 python -m pytest $T -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest.log
shift
for w in ${@:-config5}; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-ttt > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
  tail -3 gpurun_out/bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'GDoF/s frac', round(d['roofline']['cycle_frac'],3)); print({k: round(v,3) for k,v in d['kernel_ms'].items()})"
done
