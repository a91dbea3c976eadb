#!/bin/bash
# Full round check on one B200: smoke, GPU tests, default bench (+CPU leg), reference arm, sharded
# path on one rank, the other configs' bench lines, ncu launch list (+ DRAM bytes) of the default
# bench, full captures of the three finest-level kernels and of the Galerkin setup kernels.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; cat gpurun_out/bench_default.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --force-shard --steps 20 --warmup 3 > gpurun_out/bench_shard1.json 2> gpurun_out/bench_shard1.err; echo "shard1 rc=$?"; cat gpurun_out/bench_shard1.json
for w in config1 config2 config3 config4; do
  timeout 1200 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-ttt"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_config5.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python tools/traffic.py gpurun_out/launches_config5.csv config5 6 gpurun_out/traffic.json
CMD="python tools/run_cycles.py config5 3"
for kv in "k3_smc 1" "k3_up_dict 1" "k3_top4r 1" "k3_rap_y 0" "k3_rap_out 0"; do
  set -- $kv
  ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -f -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
done
