"""Host-side mesh model: the tripartitioned spacetree the engine is built from.

Mirrors the data model of the reference's ``Spacetree``
(``/root/reference/pkg/src/treemg/spacetree.py:86-332``): per level l a
boolean ``refined[l]`` of shape ``(3**l, 3**l)`` (l < lmax), a per-cell
material sample array ``eps[l]`` and a vertex field ``u[l]`` of shape
``(3**l+1, 3**l+1)``, C-ordered, ``[i, j]`` with i along x.  Any object with
these attributes (the reference's own ``Spacetree`` included) can be handed
to :class:`paper_1903_10367_b200.solvers.GpuEngine`.

This module is mesh bookkeeping only (construction and refinement, which run
between solves); the solver classifies vertices on the device
(``tmg_kinds`` kernel) from ``refined``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["VertexKind", "CellId", "EpsilonField", "constant_field", "half_domain_jump",
           "needle_inclusion", "skew_checkerboard", "epsilon_cells", "Spacetree",
           "build_regular", "dlinear_refine"]


class VertexKind:
    """Vertex classes (spacetree.py:67-72)."""
    NONE = 0
    INTERIOR_DOF = 1
    DIRICHLET = 2
    HANGING = 3
    COARSE_OVERLAPPED = 4


@dataclass(frozen=True, order=True)
class CellId:
    level: int
    i: int
    j: int

    def parent(self) -> "CellId":
        return CellId(self.level - 1, self.i // 3, self.j // 3)


@dataclass(frozen=True)
class EpsilonField:
    """Material descriptor (discretization.py:56-80): constant | half-jump | needle | skew."""
    variant: str = "constant"
    k: int = 0
    value: float = 1.0

    def __post_init__(self):
        if self.variant not in ("constant", "half-jump", "needle", "skew"):
            raise ValueError(f"unknown epsilon field variant {self.variant!r}")
        if self.variant == "constant":
            if self.value <= 0.0:
                raise ValueError("constant epsilon must be positive")
        elif not 1 <= self.k <= 5:
            raise ValueError("contrast exponent k must be in 1..5")


def constant_field(value: float = 1.0) -> EpsilonField:
    return EpsilonField("constant", value=value)


def half_domain_jump(k: int) -> EpsilonField:
    return EpsilonField("half-jump", k=k)


def needle_inclusion(k: int) -> EpsilonField:
    return EpsilonField("needle", k=k)


def skew_checkerboard(k: int) -> EpsilonField:
    return EpsilonField("skew", k=k)


def epsilon_cells(fld: EpsilonField, level: int) -> np.ndarray:
    """Midpoint samples on the (3**l, 3**l) cell grid (discretization.py:125-145)."""
    n = 3**level
    if fld.variant == "constant":
        return np.full((n, n), fld.value)
    c = (np.arange(n) + 0.5) / n
    x, y = np.meshgrid(c, c, indexing="ij")
    low = 10.0 ** (-fld.k)
    if fld.variant == "half-jump":
        return np.where(x > 0.5, low, 1.0)
    if fld.variant == "needle":
        return np.where((np.abs(x - 0.5) <= 0.01) & (y <= 0.5), 1.0, low)
    same = ((y - (5.0 * x - 2.5)) > 0.0) == ((y - (0.2 * x + 0.5)) > 0.0)
    return np.where(same, 1.0, low)


def dlinear_refine(c: np.ndarray) -> np.ndarray:
    """d-linear interpolation to the next level, axis 0 then axis 1.

    Same per-element expression as operators.py:96-127
    (``wl*c[q] + (1-wl)*c[q+1]`` with ``wl = 1 - r/3``), used for the values
    of vertices created by refinement.
    """
    def along0(a):
        m = a.shape[0] - 1
        q, r = np.divmod(np.arange(3 * m + 1), 3)
        wl = (1.0 - r / 3.0)[:, None]
        out = wl * a[q]
        out += (1.0 - wl) * a[np.minimum(q + 1, m)]
        return out
    return along0(along0(c).T).T


class Spacetree:
    """Adaptive tripartitioned mesh plus the solution field (spacetree.py:86-120).

    New level arrays carry the reference's boundary data (u = 1 on y = 0,
    spacetree.py:116-118); callers wanting homogeneous data zero ``u``.
    """

    def __init__(self, lmin: int = 1, lmax: int = 2, field: EpsilonField | None = None):
        if lmin < 1:
            raise ValueError("lmin must be at least 1")
        if lmax < lmin:
            raise ValueError("lmax must not be smaller than lmin")
        self.lmin, self.lmax = lmin, lmax
        self.field = field if field is not None else constant_field(1.0)
        self.refined = [np.zeros((3**l, 3**l), dtype=bool) for l in range(lmax)]
        self.u: list[np.ndarray] = []
        self.eps: list[np.ndarray] = []
        self._ensure_level_arrays(0)

    def _ensure_level_arrays(self, level: int) -> None:
        while len(self.u) <= level:
            l = len(self.u)
            u = np.zeros((3**l + 1, 3**l + 1))
            u[:, 0] = 1.0
            self.u.append(u)
            self.eps.append(epsilon_cells(self.field, l))

    @property
    def depth(self) -> int:
        for l in range(self.lmax - 1, -1, -1):
            if self.refined[l].any():
                return l + 1
        return 0

    def cells_exist(self, level: int) -> np.ndarray:
        if level == 0:
            return np.ones((1, 1), dtype=bool)
        return np.kron(self.refined[level - 1], np.ones((3, 3), dtype=bool))

    def adjacent_cell_count(self, level: int) -> np.ndarray:
        e = self.cells_exist(level).astype(np.int8)
        n = e.shape[0]
        cnt = np.zeros((n + 1, n + 1), dtype=np.int8)
        for di in (0, 1):
            for dj in (0, 1):
                cnt[di:di + n, dj:dj + n] += e
        return cnt

    def vertex_kinds(self, level: int) -> np.ndarray:
        """Host classification (spacetree.py:164-191); the engine recomputes it on device."""
        n = 3**level
        cnt = self.adjacent_cell_count(level)
        kinds = np.zeros((n + 1, n + 1), dtype=np.int8)
        border = np.zeros((n + 1, n + 1), dtype=bool)
        border[[0, n], :] = True
        border[:, [0, n]] = True
        kinds[(cnt > 0) & border] = VertexKind.DIRICHLET
        inner = (cnt > 0) & ~border
        kinds[inner & (cnt < 4)] = VertexKind.HANGING
        full = inner & (cnt == 4)
        if level < self.lmax:
            r = np.pad(self.refined[level].astype(np.int8), 1)
            all4 = (r[:-1, :-1] + r[1:, :-1] + r[:-1, 1:] + r[1:, 1:]) == 4
            kinds[full & all4] = VertexKind.COARSE_OVERLAPPED
            kinds[full & ~all4] = VertexKind.INTERIOR_DOF
        else:
            kinds[full] = VertexKind.INTERIOR_DOF
        return kinds

    def dof_mask(self, level: int) -> np.ndarray:
        k = self.vertex_kinds(level)
        return (k == VertexKind.INTERIOR_DOF) | (k == VertexKind.COARSE_OVERLAPPED)

    def composite_mask(self, level: int) -> np.ndarray:
        return self.vertex_kinds(level) == VertexKind.INTERIOR_DOF

    def interior_dof_count(self, level: int) -> int:
        return int(self.composite_mask(level).sum())

    def refine_many(self, cells) -> int:
        """Batched refinement, coarse levels first (spacetree.py:247-291).

        Cells at lmax are skipped, already refined cells ignored, missing
        cells raise ValueError.  New vertices get d-linear values (boundary
        data on the domain edge).  Returns the number of vertices created.
        """
        by_level: dict[int, list[CellId]] = {}
        for c in cells:
            if c.level > 0 and not self.refined[c.level - 1][c.i // 3, c.j // 3]:
                raise ValueError(f"cell {c} does not exist")
            if c.level >= self.lmax:
                continue
            by_level.setdefault(c.level, []).append(c)
        created = 0
        for l in sorted(by_level):
            self._ensure_level_arrays(l + 1)
            before = self.adjacent_cell_count(l + 1)
            todo = [c for c in by_level[l] if not self.refined[l][c.i, c.j]]
            if not todo:
                continue
            for c in todo:
                self.refined[l][c.i, c.j] = True
            born = (before == 0) & (self.adjacent_cell_count(l + 1) > 0)
            if not born.any():
                continue
            vals = dlinear_refine(self.u[l])
            n = 3 ** (l + 1)
            ii, jj = np.nonzero(born)
            on_edge = (ii == 0) | (jj == 0) | (ii == n) | (jj == n)
            self.u[l + 1][ii, jj] = np.where(on_edge, np.where(jj == 0, 1.0, 0.0), vals[ii, jj])
            created += int(born.sum())
        return created

    def refine(self, cell: CellId) -> int:
        if cell.level > 0 and not self.refined[cell.level - 1][cell.i // 3, cell.j // 3]:
            raise ValueError(f"cell {cell} does not exist")
        if cell.level < self.lmax and self.refined[cell.level][cell.i, cell.j]:
            raise ValueError(f"cell {cell} is already refined")
        return self.refine_many([cell])


def build_regular(levels: int, lmin: int = 1, lmax: int | None = None,
                  field: EpsilonField | None = None) -> Spacetree:
    """Every cell refined on levels 0..levels-1 (spacetree.py:318-332)."""
    if levels < 1:
        raise ValueError("need at least one refined level to obtain DoFs")
    tree = Spacetree(lmin=lmin, lmax=levels if lmax is None else lmax, field=field)
    for l in range(levels):
        tree.refined[l][:, :] = True
        tree._ensure_level_arrays(l + 1)
    return tree
