"""Fixtures for the 3D GPU parity tests, produced by the 3D CPU oracle (oracle/mg3d.py).

There is no 3D reference (treemg is 2D only), so these fixtures pin the GPU
path to the oracle's semantics at sizes the oracle takes minutes to run,
including depth 5 with config 5's 27-cell coefficient blocks (the case where
the device's weight dictionaries engage, i.e. the kernels the config-5 bench
line runs).  Each fixture stores

* the per-cycle ``l2h`` / ``linf`` history;
* per level: ``sum(u)``, ``sum(u*u)``, ``max|u|`` of the final iterate and a
  strided sample ``u[o::s, o::s, o::s]`` (``s = SAMPLE_STRIDE``, offset ``o``
  per level so the sample is not only coarse points), compared with the north
  star's relative 1e-10;

as ``<name>.npz`` (meta JSON inside).

    python tests/golden3d/make_golden3d.py [name ...]
"""

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from oracle import mg3d  # noqa: E402
from paper_1903_10367_b200 import workloads  # noqa: E402

SAMPLE_STRIDE = 7


CASES = {  # workload name (workloads.by_name) -> cycles
    "config3-L4": 12,
    "config5-L4": 6,
    "config5-L5b27": 4,
    "random-L5": 3,
    "config3-L5": 8,
}


def make(name):
    n = CASES[name]
    wl = workloads.by_name(name)
    t = mg3d.Tree(wl.tree.depth, wl.tree.lmin)
    t.eps[wl.tree.depth] = wl.tree.eps[wl.tree.depth].copy()
    t0 = time.time()
    e = mg3d.Engine(t, mg3d.Config(variant=wl.variant, flavor=wl.flavor))
    e.rhs.update({l: b.copy() for l, b in wl.rhs.items()})
    t1 = time.time()
    hist = [e.advance() for _ in range(n)]
    t2 = time.time()
    meta = {"workload": name, "cycles": n, "variant": wl.variant, "flavor": wl.flavor,
            "stride": SAMPLE_STRIDE, "setup_s": round(t1 - t0, 1), "cycle_s": round((t2 - t1) / n, 1)}
    arrs = {"l2h": np.array([s.l2h for s in hist]), "linf": np.array([s.linf for s in hist])}
    for l in range(wl.tree.lmin, wl.tree.depth + 1):
        u = t.u[l]
        o = l % SAMPLE_STRIDE
        arrs[f"norms_{l}"] = np.array([u.sum(), (u * u).sum(), np.abs(u).max()])
        arrs[f"sample_{l}"] = np.ascontiguousarray(u[o::SAMPLE_STRIDE, o::SAMPLE_STRIDE, o::SAMPLE_STRIDE])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), meta=json.dumps(meta), **arrs)
    print(name, meta, hist[-1].l2h / hist[0].l2h, flush=True)


def main():
    for name in (sys.argv[1:] or list(CASES)):
        make(name)


if __name__ == "__main__":
    main()
