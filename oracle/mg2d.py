"""2D CPU restatement of the treemg cycle and operator setup (TEST ORACLE).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import this.

Every function evaluates, per array element, the same fp64 expression DAG as
the reference function it cites (all paths relative to
``/root/reference/pkg/src/treemg``), so the iterates it produces equal the
reference's bit for bit wherever the reference's arithmetic is elementwise
numpy.  The only non-elementwise arithmetic, the batched 4x4 BoxMG solve, is
delegated to ``np.linalg.solve`` exactly as the reference does
(operators.py:406), and the residual norms use numpy's pairwise ``sum`` as
the reference does (solvers.py:440).

Layout follows the reference: a level with ``n = 3**l`` cells per axis holds
vertex fields as ``(n+1, n+1)`` C-ordered arrays indexed ``[i, j]`` with i
along x, cell fields as ``(n, n)``; stencil tables are ``(n+1, n+1, 3, 3)``;
prolongation / smoothed-restriction tables are ``(nc+1, nc+1, 7, 7)`` over
fine offsets -3..3.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np

# -- vertex classes (spacetree.py:67-72) ------------------------------------
NONE, INTERIOR_DOF, DIRICHLET, HANGING, OVERLAPPED = 0, 1, 2, 3, 4

VARIANTS = ("additive", "additive-exp", "bpx", "afacc", "adafac-pi",
            "adafac-jac", "multiplicative-v10")

# -- discretization constants (discretization.py:36-47) ---------------------
CORNERS = ((0, 0), (1, 0), (0, 1), (1, 1))
ELEM = np.array([
    [2.0 / 3.0, -1.0 / 6.0, -1.0 / 6.0, -1.0 / 3.0],
    [-1.0 / 6.0, 2.0 / 3.0, -1.0 / 3.0, -1.0 / 6.0],
    [-1.0 / 6.0, -1.0 / 3.0, 2.0 / 3.0, -1.0 / 6.0],
    [-1.0 / 3.0, -1.0 / 6.0, -1.0 / 6.0, 2.0 / 3.0],
])


def nine_point(eps: float) -> np.ndarray:
    """Interior 9-point stencil of a constant material (discretization.py:165-167)."""
    return eps / 3.0 * np.array([[-1.0, -1.0, -1.0], [-1.0, 8.0, -1.0], [-1.0, -1.0, -1.0]])


def dlinear_weight(a: int, b: int) -> float:
    """d-linear weight of a coarse vertex seen from fine offset (a, b) (operators.py:80-82)."""
    return max(0.0, 1.0 - abs(a) / 3.0) * max(0.0, 1.0 - abs(b) / 3.0)


def dlinear_table7() -> np.ndarray:
    """7x7 d-linear prolongation footprint (operators.py:85-89)."""
    w = np.maximum(0.0, 1.0 - np.abs(np.arange(-3, 4)) / 3.0)
    return np.outer(w, w)


# -- material fields (discretization.py:50-145) ------------------------------

@dataclass(frozen=True)
class Field:
    variant: str = "constant"   # constant | half-jump | needle | skew
    k: int = 0
    value: float = 1.0


def cell_samples(f: Field, level: int) -> np.ndarray:
    """Midpoint samples on the full (3**l, 3**l) cell grid (discretization.py:125-145)."""
    n = 3**level
    if f.variant == "constant":
        return np.full((n, n), f.value)
    mid = (np.arange(n) + 0.5) / n
    x = np.broadcast_to(mid[:, None], (n, n))
    y = np.broadcast_to(mid[None, :], (n, n))
    low = 10.0 ** (-f.k)
    if f.variant == "half-jump":
        return np.where(x > 0.5, low, 1.0)
    if f.variant == "needle":
        return np.where((np.abs(x - 0.5) <= 0.01) & (y <= 0.5), 1.0, low)
    steep = (y - (5.0 * x - 2.5)) > 0.0
    flat = (y - (0.2 * x + 0.5)) > 0.0
    return np.where(steep == flat, 1.0, low)


# -- mesh (spacetree.py) -----------------------------------------------------

class Tree:
    """Per-level dense storage of a tripartitioned spacetree (spacetree.py:86-120).

    refined[l] (l < lmax) flags refined cells of level l; u[l], eps[l] hold
    vertex values and per-cell material samples.  New level arrays carry the
    reference's boundary data u = 1 on the edge y = 0 (spacetree.py:116-118).
    """

    def __init__(self, lmin: int = 1, lmax: int = 2, fld: Field | None = None):
        self.lmin, self.lmax = lmin, lmax
        self.fld = fld or Field()
        self.refined = [np.zeros((3**l, 3**l), dtype=bool) for l in range(lmax)]
        self.u: list[np.ndarray] = []
        self.eps: list[np.ndarray] = []
        self._grow(0)

    def _grow(self, level: int) -> None:
        while len(self.u) <= level:
            l = len(self.u)
            u = np.zeros((3**l + 1, 3**l + 1))
            u[:, 0] = 1.0
            self.u.append(u)
            self.eps.append(cell_samples(self.fld, l))

    @property
    def depth(self) -> int:
        """Finest level with cells (spacetree.py:130-136)."""
        for l in range(self.lmax - 1, -1, -1):
            if self.refined[l].any():
                return l + 1
        return 0

    def cells_exist(self, l: int) -> np.ndarray:
        if l == 0:
            return np.ones((1, 1), dtype=bool)
        r = self.refined[l - 1]
        return np.repeat(np.repeat(r, 3, axis=0), 3, axis=1)

    def cell_count(self, l: int) -> np.ndarray:
        """Existing same-level cells around each vertex (spacetree.py:153-162)."""
        e = self.cells_exist(l).astype(np.int8)
        c = np.zeros((e.shape[0] + 1,) * 2, dtype=np.int8)
        for a0, a1 in CORNERS:
            c[a0:a0 + e.shape[0], a1:a1 + e.shape[1]] += e
        return c

    def kinds(self, l: int) -> np.ndarray:
        """Vertex classification (spacetree.py:164-191)."""
        n = 3**l
        cnt = self.cell_count(l)
        k = np.zeros((n + 1, n + 1), dtype=np.int8)
        on_edge = np.zeros_like(cnt, dtype=bool)
        on_edge[[0, -1], :] = True
        on_edge[:, [0, -1]] = True
        k[(cnt > 0) & on_edge] = DIRICHLET
        inner = (cnt > 0) & ~on_edge
        k[inner & (cnt < 4)] = HANGING
        full = inner & (cnt == 4)
        if l < self.lmax:
            rp = np.zeros((n + 2, n + 2), dtype=np.int8)
            rp[1:-1, 1:-1] = self.refined[l]
            all4 = (rp[:-1, :-1] + rp[1:, :-1] + rp[:-1, 1:] + rp[1:, 1:]) == 4
            k[full & all4] = OVERLAPPED
            k[full & ~all4] = INTERIOR_DOF
        else:
            k[full] = INTERIOR_DOF
        return k

    def dof_mask(self, l: int) -> np.ndarray:
        k = self.kinds(l)
        return (k == INTERIOR_DOF) | (k == OVERLAPPED)

    def refine_many(self, cells) -> None:
        """Batched refinement, coarse first, new vertices d-linear (spacetree.py:247-291)."""
        by_level: dict[int, list[tuple[int, int]]] = {}
        for (l, i, j) in cells:
            if l > 0 and not self.refined[l - 1][i // 3, j // 3]:
                raise ValueError(f"cell {(l, i, j)} does not exist")
            if l >= self.lmax:
                continue
            by_level.setdefault(l, []).append((i, j))
        for l in sorted(by_level):
            ch = l + 1
            self._grow(ch)
            before = self.cell_count(ch)
            fresh = [(i, j) for (i, j) in by_level[l] if not self.refined[l][i, j]]
            if not fresh:
                continue
            for i, j in fresh:
                self.refined[l][i, j] = True
            born = (before == 0) & (self.cell_count(ch) > 0)
            if not born.any():
                continue
            vals = prolong_dlinear(self.u[l])
            n = 3**ch
            ii, jj = np.nonzero(born)
            edge = (ii == 0) | (jj == 0) | (ii == n) | (jj == n)
            # boundary data: 1 on y == 0 (discretization.py:148-150)
            bval = np.where(jj == 0, 1.0, 0.0)
            self.u[ch][ii, jj] = np.where(edge, bval, vals[ii, jj])


def build_regular(levels: int, lmin: int = 1, lmax: int | None = None,
                  fld: Field | None = None) -> Tree:
    """Every cell refined on levels 0..levels-1 (spacetree.py:318-332)."""
    if levels < 1:
        raise ValueError("need at least one refined level to obtain DoFs")
    t = Tree(lmin, levels if lmax is None else lmax, fld)
    for l in range(levels):
        t.refined[l][:, :] = True
        t._grow(l + 1)
    return t


# -- stencil application (operators.py:143-264) -------------------------------

def _span(N: int, d: int) -> tuple[slice, slice]:
    """(destination, source) slices with source = destination + d, in range."""
    return (slice(0, N - d), slice(d, N)) if d >= 0 else (slice(-d, N), slice(0, N + d))


def apply_const(x: np.ndarray, c_eps: float) -> np.ndarray:
    """Constant 9-point stencil, zero extension, zero taps skipped (operators.py:143-161)."""
    s = nine_point(c_eps)
    out = np.zeros_like(x)
    N = x.shape[0]
    for a in range(3):
        for b in range(3):
            if s[a, b] == 0.0:
                continue
            di, si = _span(N, a - 1)
            dj, sj = _span(N, b - 1)
            out[di, dj] += s[a, b] * x[si, sj]
    return out


def apply_element(x: np.ndarray, eps: np.ndarray) -> np.ndarray:
    """Element-wise assembly on the fly: corner a outer, b inner (operators.py:178-188)."""
    n = eps.shape[0]
    out = np.zeros_like(x)
    for a, (a0, a1) in enumerate(CORNERS):
        acc = np.zeros((n, n))
        for b, (b0, b1) in enumerate(CORNERS):
            acc += ELEM[a, b] * x[b0:b0 + n, b1:b1 + n]
        out[a0:a0 + n, a1:a1 + n] += eps * acc
    return out


def element_diag(eps: np.ndarray) -> np.ndarray:
    """Assembled diagonal, corner order (operators.py:190-199)."""
    n = eps.shape[0]
    out = np.zeros((n + 1, n + 1))
    for a, (a0, a1) in enumerate(CORNERS):
        out[a0:a0 + n, a1:a1 + n] += ELEM[a, a] * eps
    return out


def assemble_table(eps: np.ndarray) -> np.ndarray:
    """Per-vertex 3x3 rows from adjacent element matrices (operators.py:251-264)."""
    n = eps.shape[0]
    t = np.zeros((n + 1, n + 1, 3, 3))
    for a, (a0, a1) in enumerate(CORNERS):
        for b, (b0, b1) in enumerate(CORNERS):
            t[a0:a0 + n, a1:a1 + n, b0 - a0 + 1, b1 - a1 + 1] += ELEM[a, b] * eps
    return t


def apply_table(x: np.ndarray, t: np.ndarray) -> np.ndarray:
    """Stored-stencil apply, taps row-major (operators.py:229-239)."""
    N = x.shape[0]
    out = np.zeros_like(x)
    for a in range(3):
        for b in range(3):
            di, si = _span(N, a - 1)
            dj, sj = _span(N, b - 1)
            out[di, dj] += t[di, dj, a, b] * x[si, sj]
    return out


class Op:
    """A level operator: 'const' / 'element' (per-cell eps) / 'table'.

    Mirrors ElementOperator's constant detection (operators.py:172-176) and
    TableOperator (operators.py:222-248).
    """

    def __init__(self, eps: np.ndarray | None = None, table: np.ndarray | None = None):
        self.eps, self.tbl = eps, table
        self.kind = "table"
        self.c = None
        if table is None:
            first = float(eps.flat[0])
            self.c = first if first > 0.0 and np.all(eps == first) else None
            self.kind = "const" if self.c is not None else "element"
        self._diag = None

    def apply(self, x: np.ndarray) -> np.ndarray:
        if self.kind == "const":
            return apply_const(x, self.c)
        if self.kind == "element":
            return apply_element(x, self.eps)
        return apply_table(x, self.tbl)

    def diag(self) -> np.ndarray:
        if self._diag is None:
            self._diag = element_diag(self.eps) if self.tbl is None else self.tbl[:, :, 1, 1]
        return self._diag

    def table(self) -> np.ndarray:
        return assemble_table(self.eps) if self.tbl is None else self.tbl


# -- d-linear transfers (operators.py:92-132) ---------------------------------

_W5 = np.array([1.0, 2.0, 3.0, 2.0, 1.0]) / 3.0


def _prolong_axis0(c: np.ndarray) -> np.ndarray:
    m = c.shape[0] - 1
    q, r = np.divmod(np.arange(3 * m + 1), 3)
    wl = (1.0 - r / 3.0)[:, None]
    out = wl * c[q]
    out += (1.0 - wl) * c[np.minimum(q + 1, m)]
    return out


def prolong_dlinear(c: np.ndarray) -> np.ndarray:
    """Axis 0 then axis 1, wl*c[q] + (1-wl)*c[q+1] (operators.py:96-127)."""
    return _prolong_axis0(_prolong_axis0(c).T).T


def _restrict_axis0(f: np.ndarray) -> np.ndarray:
    m = (f.shape[0] - 1) // 3
    out = np.zeros((m + 1,) + f.shape[1:])
    for k, off in enumerate(range(-2, 3)):
        lo = 1 if off < 0 else 0
        hi = m - 1 if off > 0 else m
        out[lo:hi + 1] += _W5[k] * f[3 * np.arange(lo, hi + 1) + off]
    return out


def restrict_dlinear(f: np.ndarray) -> np.ndarray:
    """Accumulating transpose of d-linear P, axis 0 then 1 (operators.py:111-132)."""
    return _restrict_axis0(_restrict_axis0(f).T).T


# -- operator-dependent (BoxMG) transfers (operators.py:270-437) -------------

def _gather(arr: np.ndarray, oi: int, oj: int, nc: int) -> np.ndarray:
    """arr at fine positions 3v + (oi, oj) for every coarse v, zero outside (operators.py:270-284)."""
    nf = arr.shape[0] - 1
    ii = 3 * np.arange(nc + 1) + oi
    jj = 3 * np.arange(nc + 1) + oj
    vi = (ii >= 0) & (ii <= nf)
    vj = (jj >= 0) & (jj <= nf)
    out = np.zeros((nc + 1, nc + 1) + arr.shape[2:], dtype=arr.dtype)
    out[np.ix_(vi, vj)] = arr[np.ix_(ii[vi], jj[vj])]
    return out


def _edge_weights(c1: np.ndarray, c2: np.ndarray, active: np.ndarray):
    """Closed-form 2x2 lumped solve for the two face points of an edge (operators.py:287-303)."""
    am1, a01, ap1 = c1[..., 0], c1[..., 1], c1[..., 2]
    am2, a02, ap2 = c2[..., 0], c2[..., 1], c2[..., 2]
    det = a01 * a02 - ap1 * am2
    scale = np.abs(a01 * a02) + np.abs(ap1 * am2)
    if (active & (np.abs(det) <= 1e-14 * np.maximum(scale, 1e-300))).any():
        raise ArithmeticError("degenerate collapsed stencil in face-point solve")
    det = np.where(active, det, 1.0)
    return (np.where(active, (-am1) * a02 / det, 0.0),
            np.where(active, am2 * am1 / det, 0.0),
            np.where(active, ap1 * ap2 / det, 0.0),
            np.where(active, a01 * (-ap2) / det, 0.0))


def _lump(t: np.ndarray, axis: int) -> np.ndarray:
    """Sequential 3-term sum along one stencil axis (numpy's n<8 reduction order)."""
    if axis == 3:
        return (t[..., 0] + t[..., 1]) + t[..., 2]
    return (t[..., 0, :] + t[..., 1, :]) + t[..., 2, :]


def boxmg_p(fine_tbl: np.ndarray, refined: np.ndarray, fine_kinds: np.ndarray | None) -> np.ndarray:
    """Operator-dependent prolongation weights (nc+1, nc+1, 7, 7) (operators.py:306-437)."""
    nc = refined.shape[0]
    nf = 3 * nc
    p = np.zeros((nc + 1, nc + 1, 7, 7))
    p[:, :, 3, 3] = 1.0
    # edges along x between (I,J) and (I+1,J): lump over the y taps
    act_x = np.zeros((nc, nc + 1), dtype=bool)
    act_x[:, 1:] |= refined
    act_x[:, :-1] |= refined
    ex = _edge_weights(_lump(fine_tbl[1::3, ::3], 3), _lump(fine_tbl[2::3, ::3], 3), act_x)
    # edges along y between (I,J) and (I,J+1): lump over the x taps
    act_y = np.zeros((nc + 1, nc), dtype=bool)
    act_y[1:, :] |= refined
    act_y[:-1, :] |= refined
    ey = _edge_weights(_lump(fine_tbl[::3, 1::3], 2), _lump(fine_tbl[::3, 2::3], 2), act_y)
    for (slot_lo, slot_hi, w_lo, w_hi) in ((4, 2, 0, 3), (5, 1, 1, 2)):
        # low c-point sees offset +1/+2, high c-point -2/-1
        p[:-1, :, slot_lo, 3] = np.where(act_x, ex[w_lo], p[:-1, :, slot_lo, 3])
        p[1:, :, slot_hi, 3] = np.where(act_x, ex[w_hi], p[1:, :, slot_hi, 3])
        p[:, :-1, 3, slot_lo] = np.where(act_y, ey[w_lo], p[:, :-1, 3, slot_lo])
        p[:, 1:, 3, slot_hi] = np.where(act_y, ey[w_hi], p[:, 1:, 3, slot_hi])

    ci, cj = np.nonzero(refined)
    if ci.size:
        m = ci.size
        interior = ((1, 1), (2, 1), (1, 2), (2, 2))
        corner = ((0, 0), (3, 0), (0, 3), (3, 3))
        known = np.zeros((m, 4, 4, 4))       # patch (p, q) x corner
        for c, (cp, cq) in enumerate(corner):
            known[:, cp, cq, c] = 1.0
        for q, dj in ((0, 0), (3, 1)):        # edges along x: bottom / top
            for pp, k_lo, k_hi in ((1, 0, 2), (2, 1, 3)):
                known[:, pp, q, 2 * dj] = ex[k_lo][ci, cj + dj]
                known[:, pp, q, 1 + 2 * dj] = ex[k_hi][ci, cj + dj]
        for pp, di in ((0, 0), (3, 1)):       # edges along y: left / right
            for qq, k_lo, k_hi in ((1, 0, 2), (2, 1, 3)):
                known[:, pp, qq, di] = ey[k_lo][ci + di, cj]
                known[:, pp, qq, 2 + di] = ey[k_hi][ci + di, cj]
        a_ff = np.zeros((m, 4, 4))
        rhs = np.zeros((m, 4, 4))
        for r, (fp, fq) in enumerate(interior):
            row = fine_tbl[3 * ci + fp, 3 * cj + fq]
            for da in (-1, 0, 1):
                for db in (-1, 0, 1):
                    tgt = (fp + da, fq + db)
                    coef = row[:, da + 1, db + 1]
                    if tgt in interior:
                        a_ff[:, r, interior.index(tgt)] += coef
                    else:
                        rhs[:, r, :] -= coef[:, None] * known[:, tgt[0], tgt[1], :]
        sol = np.linalg.solve(a_ff, rhs)
        for c, (cp, cq) in enumerate(corner):
            wi, wj = ci + cp // 3, cj + cq // 3
            for r, (fp, fq) in enumerate(interior):
                p[wi, wj, 3 * ci + fp - 3 * wi + 3, 3 * cj + fq - 3 * wj + 3] = sol[:, r, c]

    if fine_kinds is not None:
        hang = (fine_kinds == HANGING).astype(float)
        for oi in range(-3, 4):
            for oj in range(-3, 4):
                hit = _gather(hang, oi, oj, nc) > 0.5
                if hit.any():
                    p[:, :, oi + 3, oj + 3] = np.where(hit, dlinear_weight(oi, oj),
                                                       p[:, :, oi + 3, oj + 3])
    idx = 3 * np.arange(nc + 1)
    for o in range(-3, 4):
        out = (idx + o < 0) | (idx + o > nf)
        p[out, :, o + 3, :] = 0.0
        p[:, out, :, o + 3] = 0.0
    return p


def galerkin(fine_masked: np.ndarray, p: np.ndarray) -> np.ndarray:
    """Coarse rows of P^T A P, loop order of operators.py:446-478."""
    nc = p.shape[0] - 1
    out = np.zeros((nc + 1, nc + 1, 3, 3))
    pad = np.zeros((nc + 3, nc + 3, 7, 7))
    pad[1:-1, 1:-1] = p
    for oi in range(-2, 3):
        for oj in range(-2, 3):
            r_w = p[:, :, oi + 3, oj + 3]
            if not np.any(r_w):
                continue
            arow = _gather(fine_masked, oi, oj, nc)
            for si in (-1, 0, 1):
                for sj in (-1, 0, 1):
                    acoef = arow[:, :, si + 1, sj + 1]
                    for dwi in (-1, 0, 1):
                        pi = oi + si - 3 * dwi
                        if not -3 <= pi <= 3:
                            continue
                        for dwj in (-1, 0, 1):
                            pj = oj + sj - 3 * dwj
                            if not -3 <= pj <= 3:
                                continue
                            p_w = pad[1 + dwi:nc + 2 + dwi, 1 + dwj:nc + 2 + dwj, pi + 3, pj + 3]
                            out[:, :, dwi + 1, dwj + 1] += r_w * acoef * p_w
    return out


def rtilde_unit(omega: float) -> np.ndarray:
    """Truncated 7x7 stencil of omega R A1 diag(A1)^-1 (operators.py:484-505)."""
    r7 = dlinear_table7()
    a1 = nine_point(1.0)
    raw = np.zeros((9, 9))
    for ji in range(-3, 4):
        for jj in range(-3, 4):
            w = r7[ji + 3, jj + 3]
            if w == 0.0:
                continue
            for si in (-1, 0, 1):
                for sj in (-1, 0, 1):
                    raw[ji + si + 4, jj + sj + 4] += w * a1[si + 1, sj + 1] * (3.0 / 8.0)
    raw *= omega
    return raw[1:-1, 1:-1]


def rtilde_table(p: np.ndarray, omega: float, fine_tbl: np.ndarray | None = None,
                 fine_diag: np.ndarray | None = None) -> np.ndarray:
    """Per-coarse-vertex 7x7 smoothed restriction (operators.py:508-547)."""
    nc = p.shape[0] - 1
    out = np.zeros((nc + 1, nc + 1, 7, 7))
    a1 = nine_point(1.0)
    for ji in range(-3, 4):
        for jj in range(-3, 4):
            w = p[:, :, ji + 3, jj + 3]
            if not np.any(w):
                continue
            arow = None if fine_tbl is None else _gather(fine_tbl, ji, jj, nc)
            for si in (-1, 0, 1):
                for sj in (-1, 0, 1):
                    ti, tj = ji + si, jj + sj
                    if not (-3 <= ti <= 3 and -3 <= tj <= 3):
                        continue
                    if arow is None:
                        out[:, :, ti + 3, tj + 3] += w * (a1[si + 1, sj + 1] * (3.0 / 8.0))
                    else:
                        dg = _gather(fine_diag, ti, tj, nc)
                        dinv = np.where(dg != 0.0, 1.0 / np.where(dg == 0, 1, dg), 0.0)
                        out[:, :, ti + 3, tj + 3] += w * arow[:, :, si + 1, sj + 1] * dinv
    out *= omega
    return out


class Transfer:
    """Transfers between level l (coarse, nc = 3**l) and l+1 (operators.py:553-631)."""

    def __init__(self, nc: int, p: np.ndarray | None, rt: np.ndarray | None,
                 rt_omega: float | None = None):
        self.nc, self.p, self.rt, self.rt_omega = nc, p, rt, rt_omega

    def prolong(self, c: np.ndarray) -> np.ndarray:
        if self.p is None:
            return prolong_dlinear(c)
        nc, nf = self.nc, 3 * self.nc
        fine = np.zeros((nf + 1, nf + 1))
        idx = 3 * np.arange(nc + 1)
        for oi in range(-3, 4):
            for oj in range(-3, 4):
                w = self.p[:, :, oi + 3, oj + 3]
                if not np.any(w):
                    continue
                vi = (idx + oi >= 0) & (idx + oi <= nf)
                vj = (idx + oj >= 0) & (idx + oj <= nf)
                fine[np.ix_(idx[vi] + oi, idx[vj] + oj)] += (w * c)[np.ix_(vi, vj)]
        return fine

    def _restrict_by(self, tbl: np.ndarray, f: np.ndarray, skip_zero: bool) -> np.ndarray:
        out = np.zeros((self.nc + 1, self.nc + 1))
        for oi in range(-3, 4):
            for oj in range(-3, 4):
                w = tbl[..., oi + 3, oj + 3]
                if skip_zero and not np.any(w):
                    continue
                out += w * _gather(f, oi, oj, self.nc)
        return out

    def restrict(self, f: np.ndarray) -> np.ndarray:
        if self.p is None:
            return restrict_dlinear(f)
        return self._restrict_by(self.p, f, True)

    def restrict_smoothed(self, f: np.ndarray) -> np.ndarray:
        if self.rt is None:
            return np.zeros((self.nc + 1, self.nc + 1))
        if self.rt_omega is not None and self.p is None:
            s = apply_const(f, 1.0)
            s *= self.rt_omega * 3.0 / 8.0
            return restrict_dlinear(s)
        return self._restrict_by(self.rt, f, self.rt.ndim == 2)


# -- engine (solvers.py) -----------------------------------------------------

@dataclass
class Config:
    variant: str = "adafac-jac"
    flavor: str = "geometric"
    omega: float = 0.6
    omega_tilde: float | None = None
    omega_hat: float = 0.7
    rtilde_true_operator: bool = False
    damping_scale: float = 1.0

    @property
    def wt(self) -> float:
        return self.omega if self.omega_tilde is None else self.omega_tilde


@dataclass
class Stats:
    l2h: float
    linf: float
    dofs: int
    updates: int
    level_dofs: dict = dc_field(default_factory=dict)


class Engine:
    """Restatement of ReferenceEngine (solvers.py:129-492)."""

    def __init__(self, tree: Tree, cfg: Config):
        if cfg.variant not in VARIANTS or cfg.flavor not in ("geometric", "boxmg"):
            raise ValueError("bad config")
        self.tree, self.cfg = tree, cfg
        self.rhs: dict[int, np.ndarray] = {}
        self.rebuild()

    def rebuild(self) -> None:
        """Operator hierarchy setup (solvers.py:145-255)."""
        t, cfg = self.tree, self.cfg
        self.ltop = top = t.depth
        if top < t.lmin:
            raise ValueError("tree has no DoF-carrying level at or above lmin")
        jac = cfg.variant == "adafac-jac"
        # effective material: refined cells take the child mean (solvers.py:165-175)
        self.eff: dict[int, np.ndarray] = {}
        for l in range(top, t.lmin - 1, -1):
            e = t.eps[l].copy()
            if l < t.lmax and t.refined[l].any():
                n = 3**l
                ch = self.eff.get(l + 1, t.eps[l + 1] if l + 1 < len(t.eps) else None)
                e = np.where(t.refined[l], ch.reshape(n, 3, n, 3).mean(axis=(1, 3)), e)
            self.eff[l] = e
        self.masks, self.hw, self.rops, self.ops, self.tr = {}, {}, {}, {}, {}
        em = {}
        for l in range(t.lmin, top + 1):
            em[l] = self.eff[l] * t.cells_exist(l)
            k = t.kinds(l)
            dof = (k == INTERIOR_DOF) | (k == OVERLAPPED)
            self.masks[l] = dict(kinds=k, dof=dof, composite=k == INTERIOR_DOF,
                                 hanging=k == HANGING, exists=k != NONE,
                                 overlapped=k == OVERLAPPED, rho_src=dof | (k == HANGING))
            some = l < t.lmax and t.refined[l].any()
            self.rops[l] = Op(self.eff[l] * t.refined[l]) if some else None
            if some:
                n = 3**l
                rp = np.zeros((n + 2, n + 2), dtype=bool)
                rp[1:-1, 1:-1] = t.refined[l]
                near = rp[:-1, :-1] | rp[1:, :-1] | rp[:-1, 1:] | rp[1:, 1:]
                self.hw[l] = np.where(near, 3.0 ** -(l + 1), 3.0**-l)
            else:
                self.hw[l] = np.full((1, 1), 3.0**-l)
        if cfg.flavor == "geometric":
            for l in range(t.lmin, top + 1):
                self.ops[l] = Op(em[l])
            for l in range(t.lmin, top):
                rt, fast = (rtilde_unit(cfg.omega), cfg.omega) if jac else (None, None)
                if jac and cfg.rtilde_true_operator:
                    ftbl = assemble_table(em[l + 1]) * self.masks[l + 1]["dof"][:, :, None, None]
                    p7 = np.broadcast_to(dlinear_table7(), (3**l + 1, 3**l + 1, 7, 7))
                    rt = rtilde_table(p7, cfg.omega, ftbl, self.ops[l + 1].diag())
                    fast = None
                self.tr[l] = Transfer(3**l, None, rt, fast)
        else:
            self.ops[top] = Op(em[top])
            raw = self.ops[top].table()
            self.ptab = {}
            for l in range(top - 1, t.lmin - 1, -1):
                fk = self.masks[l + 1]["kinds"]
                p = boxmg_p(raw, t.refined[l] & t.cells_exist(l), fk)
                masked = raw * self.masks[l + 1]["dof"][:, :, None, None]
                rap = galerkin(masked, p)
                tbl = assemble_table(em[l])
                ov = self.masks[l]["kinds"] == OVERLAPPED
                tbl[ov] = rap[ov]
                self.ops[l] = Op(table=tbl)
                rt = None
                if jac:
                    if cfg.rtilde_true_operator:
                        rt = rtilde_table(p, cfg.omega, masked, self.ops[l + 1].diag())
                    else:
                        rt = rtilde_table(p, cfg.omega)
                self.tr[l] = Transfer(3**l, p, rt)
                raw = tbl
        if cfg.variant == "multiplicative-v10":
            if top - t.lmin != 1 or not all(t.refined[l].all() for l in range(top)):
                raise ValueError("the two-grid reference needs a regular two-level tree")
            self._coarse_inv = self._dense_coarse_inverse(t.lmin)

    def _dense_coarse_inverse(self, l: int):
        """Dense inverse of the coarse interior operator (solvers.py:262-276)."""
        op, dof = self.ops[l], self.masks[l]["dof"]
        idx = np.argwhere(dof)
        pos = {(int(i), int(j)): k for k, (i, j) in enumerate(idx)}
        a = np.zeros((len(idx), len(idx)))
        tbl = op.table()
        for k, (i, j) in enumerate(idx):
            s = tbl[i, j]
            for da in range(3):
                for db in range(3):
                    q = pos.get((int(i) + da - 1, int(j) + db - 1))
                    if q is not None:
                        a[k, q] += s[da, db]
        return np.linalg.inv(a), idx

    # FAS state (solvers.py:280-296)
    def update_fas_state(self) -> None:
        t = self.tree
        for l in range(self.ltop - 1, t.lmin - 1, -1):
            fk = self.masks[l + 1]["kinds"][::3, ::3]
            take = (fk == INTERIOR_DOF) | (fk == OVERLAPPED)
            t.u[l][take] = t.u[l + 1][::3, ::3][take]
        for l in range(t.lmin, self.ltop + 1):
            h = self.masks[l]["hanging"]
            if h.any():
                t.u[l][h] = prolong_dlinear(t.u[l - 1])[h]

    def _rhs(self, l: int) -> np.ndarray:
        r = self.rhs.get(l)
        return np.zeros_like(self.tree.u[l]) if r is None else r

    def _w(self, l: int) -> float:
        if self.cfg.variant == "additive-exp":
            return self.cfg.omega_hat ** (self.ltop - l)
        return self.cfg.omega

    def _bpart(self, l: int, au: np.ndarray) -> np.ndarray:
        """FAS operator image over the refined region (solvers.py:318-332)."""
        rop = self.rops[l]
        if rop is None:
            return np.zeros_like(au)
        ar = rop.apply(self.tree.u[l])
        ov = self.masks[l]["overlapped"]
        return np.where(ov, au, ar) if ov.any() else ar

    def _stats_add(self, st: Stats, l: int, r: np.ndarray) -> None:
        """solvers.py:435-443."""
        comp = self.masks[l]["composite"]
        if comp.any():
            rr = r[comp]
            h = np.broadcast_to(self.hw[l], r.shape)[comp]
            st.l2h += float(((h * rr) ** 2).sum())
            st.linf = max(st.linf, float(np.abs(rr).max()))
            st.dofs += int(comp.sum())
        st.level_dofs[l] = int(self.masks[l]["dof"].sum())

    def count_updates(self) -> int:
        """solvers.py:449-459."""
        l0, l1, v = self.tree.lmin, self.ltop, self.cfg.variant
        dof = {l: int(self.masks[l]["dof"].sum()) for l in range(l0, l1 + 1)}
        total = sum(dof.values())
        if v == "adafac-jac":
            total += sum(dof[l] for l in range(l0, l1))
        elif v == "adafac-pi":
            total += sum(dof[l] for l in range(l0 + 1, l1 + 1))
        return total

    def advance(self) -> Stats:
        """One additive cycle; stats of the starting iterate (solvers.py:334-399)."""
        if self.cfg.variant == "multiplicative-v10":
            return self._advance_v10()
        t, cfg = self.tree, self.cfg
        l0, l1 = t.lmin, self.ltop
        b = {l1: self._rhs(l1)}
        d, dt = {}, {}
        st = Stats(0.0, 0.0, 0, 0, {})
        rho_below = None
        for l in range(l1, l0 - 1, -1):
            op, m = self.ops[l], self.masks[l]
            dof = m["dof"]
            diag = np.where(dof, op.diag(), 1.0)
            au = op.apply(t.u[l])
            if l < l1:
                b[l] = b[l] + self._bpart(l, au)
            rho = np.where(m["rho_src"], b[l] - au, 0.0)
            rdof = np.where(dof, rho, 0.0)
            self._stats_add(st, l, rdof)
            if cfg.variant == "bpx" and l < l1:
                d[l] = cfg.omega * rdof
            else:
                d[l] = self._w(l) * rdof / diag
            if cfg.variant == "adafac-jac" and l < l1:
                dt[l] = cfg.damping_scale * (cfg.wt * self.tr[l].restrict_smoothed(rho_below) / diag)
                dt[l][~dof] = 0.0
            if l > l0:
                src = rho
                if cfg.variant == "afacc":
                    src = rho.copy()
                    src[::3, ::3] = 0.0
                b[l - 1] = self.tr[l - 1].restrict(src)
                b[l - 1] += self._rhs(l - 1)
            rho_below = rdof
        if cfg.variant == "adafac-pi":
            for l in range(l0 + 1, l1 + 1):
                inj = np.zeros_like(t.u[l - 1])
                fk = self.masks[l]["kinds"][::3, ::3]
                take = (fk == INTERIOR_DOF) | (fk == OVERLAPPED)
                inj[take] = d[l][::3, ::3][take]
                dt[l] = cfg.damping_scale * self.tr[l - 1].prolong(inj)
                dt[l][~self.masks[l]["dof"]] = 0.0
        carry = None
        for l in range(l0, l1 + 1):
            g = d[l] - dt[l] if l in dt else d[l]
            carry = g if carry is None else self.tr[l - 1].prolong(carry) + g
            carry[~self.masks[l]["exists"]] = 0.0
            t.u[l] += carry
        self.update_fas_state()
        st.updates = self.count_updates()
        st.l2h = float(np.sqrt(st.l2h))
        return st

    def _advance_v10(self) -> Stats:
        """Two-grid V(1,0) reference (solvers.py:401-428)."""
        t, cfg = self.tree, self.cfg
        l0, l1 = t.lmin, self.ltop
        opf = self.ops[l1]
        dof_f, dof_c = self.masks[l1]["dof"], self.masks[l0]["dof"]
        st = Stats(0.0, 0.0, 0, 0, {})
        rho = np.where(dof_f, self._rhs(l1) - opf.apply(t.u[l1]), 0.0)
        self._stats_add(st, l1, rho)
        self._stats_add(st, l0, np.where(dof_c, self.tr[l0].restrict(rho), 0.0))
        t.u[l1] += cfg.omega * rho / np.where(dof_f, opf.diag(), 1.0)
        self.update_fas_state()
        rho_sm = np.where(dof_f, self._rhs(l1) - opf.apply(t.u[l1]), 0.0)
        rho_c = np.where(dof_c, self.tr[l0].restrict(rho_sm), 0.0)
        inv, idx = self._coarse_inv
        c = np.zeros_like(t.u[l0])
        c[tuple(idx.T)] = inv @ rho_c[tuple(idx.T)]
        t.u[l0] += c
        t.u[l1] += self.tr[l0].prolong(c)
        self.update_fas_state()
        st.updates = self.count_updates()
        st.l2h = float(np.sqrt(st.l2h))
        return st

    def residual_stats(self) -> Stats:
        """Residual of the current iterate, no update (solvers.py:461-482)."""
        t = self.tree
        l0, l1 = t.lmin, self.ltop
        b = {l1: self._rhs(l1)}
        st = Stats(0.0, 0.0, 0, 0, {})
        for l in range(l1, l0 - 1, -1):
            au = self.ops[l].apply(t.u[l])
            if l < l1:
                b[l] = b[l] + self._bpart(l, au)
            rho = np.where(self.masks[l]["rho_src"], b[l] - au, 0.0)
            self._stats_add(st, l, np.where(self.masks[l]["dof"], rho, 0.0))
            if l > l0:
                src = rho
                if self.cfg.variant == "afacc":
                    src = rho.copy()
                    src[::3, ::3] = 0.0
                b[l - 1] = self.tr[l - 1].restrict(src) + self._rhs(l - 1)
        st.l2h = float(np.sqrt(st.l2h))
        return st
