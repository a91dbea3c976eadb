"""Host-side mesh model for 3D regular tripartitioned spacetrees (configs 3, 5).

The reference's data model (``spacetree.py:86-120``) carried to d = 3 for
regular trees: levels 0..depth, every cell of levels < depth refined,
``u[l]`` of shape ``(3**l+1,)*3`` and ``eps[l]`` of shape ``(3**l,)*3``,
C-ordered ``[i, j, k]`` with i along x.  Only the finest level's ``eps`` is
material input (coarser materials are child means, computed on the device).
"""

from __future__ import annotations

import numpy as np

from .spacetree import VertexKind

__all__ = ["Spacetree3", "build_regular3"]


class Spacetree3:
    def __init__(self, levels: int, lmin: int = 1):
        if levels < 1:
            raise ValueError("need at least one refined level to obtain DoFs")
        if lmin < 1 or lmin > levels:
            raise ValueError("lmin must lie in [1, levels]")
        self.lmin, self.lmax = lmin, levels
        self.u = [np.zeros((3**l + 1,) * 3) for l in range(levels + 1)]
        self.eps = [np.ones((3**l,) * 3) for l in range(levels + 1)]

    dim = 3

    @property
    def depth(self) -> int:
        return self.lmax

    def vertex_kinds(self, l: int) -> np.ndarray:
        N = 3**l + 1
        k = np.full((N, N, N), VertexKind.DIRICHLET, dtype=np.int8)
        k[1:-1, 1:-1, 1:-1] = (VertexKind.COARSE_OVERLAPPED if l < self.depth
                               else VertexKind.INTERIOR_DOF)
        return k

    def kinds(self, l: int) -> np.ndarray:
        return self.vertex_kinds(l)


def build_regular3(levels: int, lmin: int = 1) -> Spacetree3:
    return Spacetree3(levels, lmin)
