#!/bin/bash
python -m paper_1903_10367_b200.build > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity3d.py -m gpu -x -q > gpurun_out/pytest_sh.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sh.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --force-shard --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_shard1.json 2> gpurun_out/bench_shard1.err; echo "shard1 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_shard1.json')); print(d['ms_per_step'], d.get('kernel_ms'))"
