"""Run a few cycles of a workload under TMG_FFP (for compute-sanitizer / quick checks):
python tools/ffp_probe.py config5-L4 3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1903_10367_b200 import GpuEngine, SolverConfig, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config5-L4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = workloads.by_name(name)
eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
eng.rhs.update(wl.rhs)
h = eng.advance_many(n)
print(name, [s.l2h for s in h])
