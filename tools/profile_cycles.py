"""Run a workload's cycle repeatedly (for ncu launch lists / full captures).

    python tools/profile_cycles.py [workload] [cycles]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1903_10367_b200 import GpuEngine, SolverConfig, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = workloads.by_name(name)
eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
eng.rhs.update(wl.rhs)
h = eng.advance_many(n)
print(name, "cycles", n, "l2h[-1]", h[-1].l2h, "launches/cycle", eng.launches_per_cycle())
