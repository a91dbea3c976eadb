"""Load golden fixtures (made by tests/golden/make_golden.py from the reference)."""

from __future__ import annotations

import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Case:
    def __init__(self, path: str):
        self.name = os.path.splitext(os.path.basename(path))[0]
        z = np.load(path)
        self.z = {k: z[k] for k in z.files}
        self.meta = json.loads(str(self.z["meta"]))

    def __getitem__(self, k):
        return self.z[k]

    def has(self, k):
        return k in self.z

    @property
    def cfg(self) -> dict:
        return dict(self.meta["cfg"])

    def levels_with(self, prefix: str):
        return sorted(int(k[len(prefix):]) for k in self.z if k.startswith(prefix)
                      and k[len(prefix):].isdigit())

    def build_tree(self, tree_cls):
        """Rebuild the case's tree in any implementation with the reference data model."""
        m = self.meta
        t = tree_cls(lmin=m["lmin"], lmax=m["lmax"])
        t.refined = [self.z[f"refined_{l}"].copy() for l in range(m["lmax"])]
        t.u = [self.z[f"u0_{l}"].copy() for l in range(m["nlev_arrays"])]
        t.eps = [self.z[f"eps_{l}"].copy() for l in range(m["nlev_arrays"])]
        return t

    def rhs(self) -> dict:
        return {l: self.z[f"rhs_{l}"].copy() for l in self.levels_with("rhs_")}


def full_cases():
    return [p for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))
            if json.loads(str(np.load(p)["meta"]))["store_u"] == "all"]


def case_names(full_only=True):
    paths = full_cases() if full_only else sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))
    return [os.path.splitext(os.path.basename(p))[0] for p in paths]


def load(name: str) -> Case:
    return Case(os.path.join(GOLDEN, name + ".npz"))
