"""Print per-phase durations of the coarse-chain kernel (diagnostics)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_10367_b200 import GpuEngine, SolverConfig, _abi, workloads  # noqa: E402

wl = workloads.by_name(sys.argv[1] if len(sys.argv) > 1 else "config2")
eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
eng.rhs.update(wl.rhs)
L = _abi.lib()
for rep in range(3):
    eng.advance_many(5)
    st = np.zeros(64, dtype=np.uint64)
    L.tmg_debug_stamps(eng._h, C.c_void_p(st.ctypes.data), 64)
    n = int(np.argmax(st == 0)) if (st == 0).any() else 64
    d = np.diff(st[:n].astype(np.int64)) / 1e3
    print("phase us:", np.round(d, 2), "total", round(float(d.sum()), 2))
