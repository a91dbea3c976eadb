"""Dynamic refinement between cycles for the GPU engine.

Host-side control plane of the reference's regrid step (``treemg/amr.py:58-171``
driven from ``treemg/bench.py:206-219``): after a cycle the iterate is pulled
from the device, cells are marked on the host, the tree is refined
(``Spacetree.refine_many``) and the engine rebuilds its hierarchy on the device
(``GpuEngine.rebuild`` + ``update_fas_state``).  The marking is restated here on
whole-level boolean masks instead of the reference's per-vertex / per-cell
Python sets; the marked cells are the same sets (tests compare whole AMR runs
against the reference's CSVs: identical DoF counts and regrid cycles).

Two criteria, as in the reference:

* boundary: every existing, unrefined cell touching the heated edge ``y = 0``
  (``j == 0``) below the depth cap, on cycles ``n % boundary_cadence == 0``
  (``amr.py:58-71``);
* curvature: per composite vertex the largest absolute axis-aligned second
  difference of ``u`` scaled by ``1 / h^2`` (same-level neighbours only,
  ``amr.py:74-99``); vertices above the lower edge of the histogram bin in
  which the top ``decile`` of the composite vertex count is reached (64 bins
  over ``(0, max]``, whole bins from the top, ``amr.py:102-151``) mark their
  adjacent existing unrefined cells (``amr.py:154-164``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .spacetree import CellId, Spacetree, VertexKind

__all__ = ["RefinePolicy", "RegridReport", "boundary_cells", "curvature_indicator", "curvature_vertices",
           "cells_around", "regrid", "marks_for_cycle"]


@dataclass(frozen=True)
class RefinePolicy:
    boundary_cadence: int = 2
    decile: float = 0.10
    bins: int = 64

    def __post_init__(self):
        if not 0.0 < self.decile < 1.0:
            raise ValueError("decile must lie in (0, 1)")
        if self.boundary_cadence < 1:
            raise ValueError("boundary cadence must be positive")


@dataclass
class RegridReport:
    refined_cells: int
    created_vertices: int

    @property
    def changed(self) -> bool:
        return self.refined_cells > 0


def _empty_marks(tree: Spacetree) -> dict[int, np.ndarray]:
    return {l: np.zeros((3**l, 3**l), dtype=bool) for l in range(min(tree.depth, tree.lmax - 1) + 1)}


def boundary_cells(tree: Spacetree, cycle: int, policy: RefinePolicy = RefinePolicy()) -> dict[int, np.ndarray]:
    """Cell masks per level: leaf cells with a face on ``y = 0`` (amr.py:58-71)."""
    marks = _empty_marks(tree)
    if cycle % policy.boundary_cadence != 0:
        return marks
    for l, m in marks.items():
        m[:, 0] = tree.cells_exist(l)[:, 0] & ~tree.refined[l][:, 0]
    return marks


def curvature_indicator(tree: Spacetree, level: int) -> np.ndarray:
    """max over the axes of |u[v-e] - 2 u[v] + u[v+e]| / h^2 where all three vertices exist."""
    u = tree.u[level]
    ex = tree.vertex_kinds(level) != VertexKind.NONE
    ind = np.zeros_like(u)
    for ax in (0, 1):
        lo = [slice(None)] * 2
        mid = [slice(None)] * 2
        hi = [slice(None)] * 2
        lo[ax], mid[ax], hi[ax] = slice(None, -2), slice(1, -1), slice(2, None)
        lo, mid, hi = tuple(lo), tuple(mid), tuple(hi)
        d2 = np.abs(u[lo] - 2.0 * u[mid] + u[hi])
        ok = ex[lo] & ex[mid] & ex[hi]
        ind[mid] = np.maximum(ind[mid], np.where(ok, d2, 0.0))
    return ind * float(9.0**level)


def curvature_vertices(tree: Spacetree, policy: RefinePolicy = RefinePolicy()) -> dict[int, np.ndarray]:
    """Vertex masks per level: composite vertices in the top bins of the indicator (amr.py:102-151)."""
    levels = range(tree.lmin, tree.depth + 1)
    scale = max([1.0] + [float(np.abs(tree.u[l]).max()) for l in levels])
    inds, comps, positive, total = {}, {}, [], 0
    for l in levels:
        comp = tree.composite_mask(l)
        ind = np.where(comp, curvature_indicator(tree, l), 0.0)
        ind[ind <= 1e-12 * scale * 9.0**l] = 0.0  # second-difference round-off never marks
        inds[l], comps[l] = ind, comp
        total += int(comp.sum())
        v = ind[comp]
        positive.append(v[v > 0.0])
    none = {l: np.zeros_like(comps[l]) for l in levels}
    vals = np.concatenate(positive) if positive else np.zeros(0)
    if total == 0 or vals.size == 0:
        return none
    top = float(vals.max())
    edges = np.linspace(0.0, top, policy.bins + 1)
    counts, _ = np.histogram(vals, bins=edges)
    # whole bins from the top until the decile of the composite vertex count is covered
    from_top = np.cumsum(counts[::-1])
    reached = np.nonzero(from_top >= policy.decile * total)[0]
    cut = policy.bins - 1 - int(reached[0]) if reached.size else 0
    threshold = edges[cut]
    return {l: comps[l] & (inds[l] > (threshold if threshold > 0.0 else 0.0)) for l in levels}


def cells_around(tree: Spacetree, vertices: dict[int, np.ndarray]) -> dict[int, np.ndarray]:
    """Existing, unrefined cells adjacent to the marked vertices, below the depth cap (amr.py:154-164)."""
    marks = _empty_marks(tree)
    for l, vm in vertices.items():
        if l >= tree.lmax or l not in marks or not vm.any():
            continue
        n = 3**l
        touched = vm[:n, :n] | vm[1:, :n] | vm[:n, 1:] | vm[1:, 1:]
        marks[l] |= touched & tree.cells_exist(l) & ~tree.refined[l]
    return marks


def marks_for_cycle(tree: Spacetree, cycle: int, policy: RefinePolicy = RefinePolicy()) -> dict[int, np.ndarray]:
    """The cells the reference's loop refines after cycle ``cycle`` (bench.py:206-209): boundary
    and curvature marks on cadence cycles, nothing otherwise."""
    marks = boundary_cells(tree, cycle, policy)
    if cycle % policy.boundary_cadence == 0:
        for l, m in cells_around(tree, curvature_vertices(tree, policy)).items():
            marks[l] |= m
    return marks


def regrid(tree: Spacetree, marks: dict[int, np.ndarray]) -> RegridReport:
    """Refine the marked cells, coarse levels first (amr.py:167-171)."""
    todo = []
    for l in sorted(marks):
        if l >= tree.lmax:
            continue
        ii, jj = np.nonzero(marks[l] & ~tree.refined[l])
        todo.extend(CellId(l, int(i), int(j)) for i, j in zip(ii, jj))
    made = tree.refine_many(todo) if todo else 0
    return RegridReport(len(todo), made)
