"""Run a few cycles of a workload on cuda:0 (for ncu captures): python tools/run_cycles.py config5 4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1903_10367_b200 import GpuEngine, SolverConfig, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
t0 = time.time()
wl = workloads.by_name(name)
t1 = time.time()
eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
eng.rhs.update(wl.rhs)
t2 = time.time()
h = eng.advance_many(n)
t3 = time.time()
print(f"{name}: inputs {t1 - t0:.1f}s setup {t2 - t1:.1f}s {n} cycles {t3 - t2:.2f}s "
      f"l2h {h[0].l2h:.6e} -> {h[-1].l2h:.6e}")
