#!/bin/bash
# Full round check on one B200: smoke, GPU tests, default bench (+CPU leg), reference arm,
# sharded path on one rank, ncu launch list of the default bench.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; cat gpurun_out/bench_default.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --force-shard --steps 20 --warmup 3 > gpurun_out/bench_shard1.json 2> gpurun_out/bench_shard1.err; echo "shard1 rc=$?"; cat gpurun_out/bench_shard1.json
python bench.py --workload config2 > gpurun_out/bench_config2.json 2> gpurun_out/bench_config2.err; echo "c2 rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_config5.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python tools/traffic.py gpurun_out/launches_config5.csv config5 6 gpurun_out/traffic.json
