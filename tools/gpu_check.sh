#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench line, ncu launch list and a
# full capture of the top kernel.  Usage (from repo root, on the GPU box):
#   bash tools/gpu_check.sh [workload] [kernel-regex]
set -u
WL=${1:-config2}
KRE=${2:-k_down}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
python bench.py --workload $WL > gpurun_out/bench_$WL.json 2> gpurun_out/bench_$WL.err; echo "bench rc=$?"
cat gpurun_out/bench_$WL.json
CMD="python bench.py --workload $WL --steps 3 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$WL.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 20 -c 3 -o gpurun_out/prof_$WL $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
