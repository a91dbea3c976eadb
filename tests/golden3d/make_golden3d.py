"""Fixtures for the 3D GPU parity tests, produced by the 3D CPU oracle.

There is no 3D reference (treemg is 2D only), so these fixtures pin the GPU
path to the oracle's semantics at sizes the oracle takes longer to run:
per-cycle l2h / linf and the SHA-256 of the final iterate on every level.

    python tests/golden3d/make_golden3d.py
"""

import hashlib
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

CASES = [("config3-L4", lambda: workloads.config3(levels=4, cycles=12), 12),
         ("config5-L4", lambda: workloads.by_name("config5-L4"), 6)]


def main():
    for name, mk, n in CASES:
        wl = mk()
        t = mg3d.Tree(wl.tree.depth, wl.tree.lmin)
        t.eps[wl.tree.depth] = wl.tree.eps[wl.tree.depth].copy()
        e = mg3d.Engine(t, mg3d.Config(variant=wl.variant, flavor=wl.flavor))
        e.rhs.update({l: b.copy() for l, b in wl.rhs.items()})
        t0 = time.time()
        hist = [e.advance() for _ in range(n)]
        out = {"workload": name if name != "config3-L4" else "config3-L4", "cycles": n,
               "variant": wl.variant, "flavor": wl.flavor,
               "l2h": [s.l2h for s in hist], "linf": [s.linf for s in hist],
               "u_sha256": {str(l): hashlib.sha256(np.ascontiguousarray(t.u[l]).tobytes()).hexdigest()
                            for l in range(wl.tree.lmin, wl.tree.depth + 1)}}
        json.dump(out, open(os.path.join(HERE, name + ".json"), "w"), indent=1)
        print(name, f"{time.time() - t0:.1f}s", hist[-1].l2h / hist[0].l2h)


if __name__ == "__main__":
    main()
