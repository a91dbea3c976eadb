"""Probe: a config-5-structured depth-5 engine with weight dictionaries, a few cycles."""
import sys

from paper_1903_10367_b200 import GpuEngine, SolverConfig, workloads

lv = int(sys.argv[1]) if len(sys.argv) > 1 else 5
wl = workloads.config5(levels=lv, block=3 ** (lv - 2))
eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
eng.rhs.update(wl.rhs)
print(eng.weight_storage(lv - 1), flush=True)
h = eng.advance_many(3)
print([s.l2h for s in h])
