"""Host vs device time of the sharded cycle on one rank (diagnostic).

    torchrun --nproc-per-node 1 tools/shard_overhead.py [workload] [cycles]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1903_10367_b200 import GpuEngine, SolverConfig, sharding, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
wl = workloads.by_name(name)
pl = sharding.plan(wl.tree.depth, 1)
eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
eng.rhs.update(wl.rhs)
eng._flush_rhs()
sh = sharding.GpuShard(eng, pl, 0)
for label, tr in (("nccl", sharding.DistTransport(pl, 0)), ("local", sharding.LocalTransport(pl))):
    se = sharding.ShardedEngine3([sh], tr, wl.variant)
    with torch.cuda.stream(sh.stream):
        for _ in range(3):
            se.cycle()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(sh.stream)
        t0 = time.perf_counter()
        for _ in range(n):
            se.cycle()
        t_host = time.perf_counter() - t0
        e1.record(sh.stream)
        torch.cuda.synchronize()
        t_all = time.perf_counter() - t0
    print(f"{label}: host enqueue {1e3 * t_host / n:.3f} ms/cycle, device {e0.elapsed_time(e1) / n:.3f} "
          f"ms/cycle, wall {1e3 * t_all / n:.3f} ms/cycle", flush=True)
