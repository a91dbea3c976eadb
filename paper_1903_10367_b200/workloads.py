"""Seeded synthetic inputs for the BASELINE configurations (2D).

The reference publishes no dataset; BASELINE.json's configs are reproduced
with seeded synthetic inputs:

* homogeneous Dirichlet data and u0 = 0 on every level;
* ``rng = np.random.default_rng(seed)``; the per-block material (if any) is
  drawn first, then the load;
* load ``rhs[l] = h_l*h_l * f`` on the composite DoFs (INTERIOR_DOF vertices)
  of every level l that has any, ``h_l = 3.0**-l``, with ``f`` iid
  U[-1, 1] drawn level by level (coarse to fine), C-order within a level; 0
  elsewhere.  (On regular trees only the finest level has composite DoFs.)

Every builder returns a :class:`Workload` whose ``tree`` is a product
:class:`~paper_1903_10367_b200.spacetree.Spacetree`; tests convert it into a
reference / oracle tree with the same ``refined``, ``eps`` and ``u`` arrays.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np

from .spacetree import CellId, Spacetree, VertexKind, build_regular
from .spacetree3d import Spacetree3

__all__ = ["Workload", "config1", "config2", "config3", "config4", "config5", "annulus_tree",
           "seeded_rhs", "random_l5", "by_name"]


@dataclass
class Workload:
    name: str
    tree: Spacetree
    variant: str
    flavor: str
    cycles: int
    target: float | None
    rhs: dict = dc_field(default_factory=dict)
    seed: int = 0

    @property
    def ltop(self) -> int:
        return self.tree.depth

    def fine_dofs(self) -> int:
        """N_fine: composite DoFs of the finest level (the metric's numerator)."""
        if getattr(self.tree, "dim", 2) == 3:
            return (3**self.ltop - 1) ** 3
        return int((self.tree.vertex_kinds(self.ltop) == VertexKind.INTERIOR_DOF).sum())

    @property
    def dim(self) -> int:
        return getattr(self.tree, "dim", 2)


def _zero_u(tree: Spacetree) -> None:
    for l in range(len(tree.u)):
        tree.u[l][:] = 0.0


def seeded_rhs(tree: Spacetree, rng: np.random.Generator) -> dict:
    out = {}
    for l in range(tree.lmin, tree.depth + 1):
        comp = tree.vertex_kinds(l) == VertexKind.INTERIOR_DOF
        cnt = int(comp.sum())
        if cnt == 0:
            continue
        f = rng.uniform(-1.0, 1.0, cnt)
        h = 3.0 ** -l
        b = np.zeros_like(tree.u[l])
        b[comp] = (h * h) * f
        out[l] = b
    return out


def config1(levels: int = 5, seed: int = 0, cycles: int = 50) -> Workload:
    """2D Poisson, eps = 1, regular depth 5, additive FAC, d-linear (BASELINE configs[0])."""
    tree = build_regular(levels)
    _zero_u(tree)
    rng = np.random.default_rng(seed)
    return Workload(f"c1-poisson-L{levels}-additive-geometric", tree, "additive", "geometric",
                    cycles, None, seeded_rhs(tree, rng), seed)


def config2(levels: int = 6, block: int | None = None, seed: int = 0,
            cycles: int = 200, target: float = 1e-8) -> Workload:
    """2D adaFACx + BoxMG/Galerkin, eps log-uniform in [1e-2, 1e2] per 27x27-cell block.

    BASELINE configs[1].  ``block`` (cells per block side) defaults to
    27 at depth 6 and scales as 3**(levels-3) so smaller depths keep 27x27
    blocks of the domain.
    """
    tree = build_regular(levels)
    _zero_u(tree)
    rng = np.random.default_rng(seed)
    n = 3**levels
    blk = block if block is not None else 3 ** max(levels - 3, 0)
    nb = n // blk
    blocks = 10.0 ** rng.uniform(-2.0, 2.0, (nb, nb))
    tree.eps[levels] = np.kron(blocks, np.ones((blk, blk)))
    return Workload(f"c2-blocks-L{levels}-adafacjac-boxmg", tree, "adafac-jac", "boxmg",
                    cycles, target, seeded_rhs(tree, rng), seed)


def annulus_tree(base: int = 4, lmax: int = 8, r_in: float = 0.20, r_out: float = 0.25,
                 centre: tuple[float, float] = (0.5, 0.5)) -> Spacetree:
    """Regular to ``base``, then refine (coarse first) every existing unrefined cell whose
    closed square meets the closed annulus ``r_in <= |x - centre| <= r_out``.

    Intersection test in fp64: ``dmin <= r_out and dmax >= r_in`` with dmin /
    dmax the nearest / farthest point of the cell square from ``centre``.
    """
    tree = build_regular(base, lmax=lmax)
    cx, cy = centre
    for l in range(base, lmax):
        n = 3**l
        lo = np.arange(n) / n
        hi = (np.arange(n) + 1) / n
        nx = np.maximum(np.maximum(lo - cx, 0.0), cx - hi)
        ny = np.maximum(np.maximum(lo - cy, 0.0), cy - hi)
        fx = np.maximum(np.abs(lo - cx), np.abs(hi - cx))
        fy = np.maximum(np.abs(lo - cy), np.abs(hi - cy))
        dmin = np.sqrt(nx[:, None] ** 2 + ny[None, :] ** 2)
        dmax = np.sqrt(fx[:, None] ** 2 + fy[None, :] ** 2)
        hit = (dmin <= r_out) & (dmax >= r_in)
        cand = hit & tree.cells_exist(l) & ~tree.refined[l]
        ii, jj = np.nonzero(cand)
        tree.refine_many([CellId(l, int(i), int(j)) for i, j in zip(ii, jj)])
    return tree


def disc_eps(level: int, inside: float = 100.0, radius: float = 0.2,
             centre: tuple[float, float] = (0.5, 0.5)) -> np.ndarray:
    n = 3**level
    mid = (np.arange(n) + 0.5) / n
    r = np.sqrt((mid[:, None] - centre[0]) ** 2 + (mid[None, :] - centre[1]) ** 2)
    return np.where(r < radius, inside, 1.0)


def config4(base: int = 4, lmax: int = 8, seed: int = 0, cycles: int = 200,
            target: float = 1e-8) -> Workload:
    """2D static annulus refinement base -> lmax, eps = 100 inside r < 0.2 (BASELINE configs[3])."""
    tree = annulus_tree(base, lmax)
    for l in range(len(tree.eps)):
        tree.eps[l] = disc_eps(l)
    _zero_u(tree)
    rng = np.random.default_rng(seed)
    return Workload(f"c4-annulus-{base}to{lmax}-adafacjac-boxmg", tree, "adafac-jac", "boxmg",
                    cycles, target, seeded_rhs(tree, rng), seed)


def seeded_rhs3(tree: Spacetree3, rng: np.random.Generator) -> dict:
    """b = h^3 f on the interior vertices of the finest level (the only composite DoFs)."""
    L = tree.depth
    n = 3**L
    f = rng.uniform(-1.0, 1.0, (n - 1,) * 3)
    h = 3.0 ** -L
    b = np.zeros((n + 1,) * 3)
    b[1:-1, 1:-1, 1:-1] = (h * h * h) * f
    return {L: b}


def config3(levels: int = 5, seed: int = 0, cycles: int = 100) -> Workload:
    """3D Poisson, eps = 1, regular depth 5, adaFACx, d-linear (BASELINE configs[2])."""
    tree = Spacetree3(levels)
    rng = np.random.default_rng(seed)
    return Workload(f"c3-poisson3d-L{levels}-adafacjac-geometric", tree, "adafac-jac", "geometric",
                    cycles, None, seeded_rhs3(tree, rng), seed)


def config5(levels: int = 6, block: int | None = None, seed: int = 0, cycles: int = 20) -> Workload:
    """3D adaFACx + BoxMG, eps log-uniform in [1e-2, 1e2] per 27^3-cell block (BASELINE configs[4]).

    ``block`` defaults to 27 cells at depth 6 and scales as 3**(levels-3), so
    smaller depths keep 27^3 blocks of the domain.
    """
    tree = Spacetree3(levels)
    rng = np.random.default_rng(seed)
    n = 3**levels
    blk = block if block is not None else 3 ** max(levels - 3, 0)
    nb = n // blk
    blocks = 10.0 ** rng.uniform(-2.0, 2.0, (nb, nb, nb))
    eps = np.empty((n, n, n))
    eps.reshape(nb, blk, nb, blk, nb, blk)[...] = blocks[:, None, :, None, :, None]
    tree.eps[levels] = eps
    return Workload(f"c5-blocks3d-L{levels}-adafacjac-boxmg", tree, "adafac-jac", "boxmg",
                    cycles, None, seeded_rhs3(tree, rng), seed)


def random_l5(seed: int = 7) -> Workload:
    """Depth-5 3D BoxMG with per-cell log-uniform coefficients: no weight row repeats, so the
    device keeps its dense weight streams (the dictionaries do not engage)."""
    wl = config5(levels=5)
    rng = np.random.default_rng(seed)
    wl.tree.eps[5][...] = 10.0 ** rng.uniform(-2, 2, wl.tree.eps[5].shape)
    wl.name = "random-L5"
    return wl


def by_name(name: str) -> Workload:
    table = {
        "config1": config1, "config2": config2, "config4": config4,
        "config2-small": lambda: config2(levels=4, cycles=30),
        "config4-small": lambda: config4(base=2, lmax=5, cycles=30),
        "config3": config3, "config5": config5,
        "config3-small": lambda: config3(levels=3, cycles=30),
        "config5-small": lambda: config5(levels=3, cycles=10),
        "config5-L4": lambda: config5(levels=4, cycles=10),
        "config3-L4": lambda: config3(levels=4, cycles=12),
        "config5-L5": lambda: config5(levels=5, cycles=10),
        "config3-L5": lambda: config3(levels=5),
        # config 5's 27-cell coefficient blocks at depth 5 (9 level-4 cells): the weight
        # dictionaries of the config-5 path engage
        "config5-L5b27": lambda: config5(levels=5, block=27),
        "random-L5": random_l5,
    }
    if name not in table:
        raise ValueError(f"unknown workload {name!r}; choose from {sorted(table)}")
    return table[name]()
