"""3D CPU restatement of the treemg cycle and operator setup (TEST ORACLE).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import this.

**Parity unpinned by the reference.**  The reference (``treemg``) is 2D only
(``SPEC.md:8``, ``SPEC.md:82``, ``SPEC.md:91``); BASELINE configs 3 and 5 are
3D.  This module is the d-generic restatement SURVEY.md §8(c) asks for: the
cycle, FAS, setup flow and every transfer are the reference's 2D algorithm
(``solvers.py:145-255``, ``:280-399``, ``:435-459``; ``operators.py:96-137``,
``:143-264``, ``:287-478``, ``:484-631``) carried to d = 3, with the 3D
decisions SURVEY.md Appendix B leaves to the builder fixed here, each with its
fp64 expression DAG (the CUDA kernels evaluate the same DAG, so the GPU path
is compared with this module bit for bit).  It is pinned by
``tests/test_oracle3d.py``:

* structure: the cycle code is the same as ``mg2d.Engine.advance`` (the
  d-generic part) -- a 2D run of ``mg2d`` equals the reference bitwise;
* a scipy sparse Galerkin FE assembly of -div(eps grad u) with trilinear
  elements (Gauss quadrature) at l <= 3: operator apply, diagonal, stencil
  tables;
* invariants restated in 3D: R == P^T (d-linear and BoxMG), RAP == P^T A P
  (dense), BoxMG P == trilinear for constant eps and reproduces constants,
  c-point rows are unit, the exact discrete solution is a fixed point of
  every variant, the cycle converges on Poisson.

3D decisions:

* regular trees only (configs 3, 5): every cell of levels < depth refined;
  vertex kinds DIRICHLET on the boundary, COARSE_OVERLAPPED inside levels
  < depth, INTERIOR_DOF inside the finest level; no hanging vertices.
* trilinear element, stiffness ``h * K_unit`` (K_unit: 1/3 diagonal, 0 for
  corners differing in one axis, -1/12 for two or three); the operator
  coefficient of a cell is ``e = eff_eps * h``.
* element apply at vertex v (ElementOperator analogue, operators.py:178-188):
  cells c = v - a in corner order a = a0 + 2 a1 + 4 a2;
  ``E = sum_a e_c`` and ``T = sum_a e_c * s_c`` sequentially from the first
  term, with ``s_c = ((x[v+(s0,s1,0)] + x[v+(s0,0,s2)]) + x[v+(0,s1,s2)]) +
  x[v+s]``, ``s = 1 - 2a``; ``A x = ((K_D*E)*x_v) - (K_E*T)``; diag ``K_D*E``.
* constant-material apply (operators.py:143-161 analogue, zero-extended):
  ``((m*x_v) - (se*SE)) - (sc*SC)`` with ``m = c*(8/3)``, ``se = c*(1/6)``,
  ``sc = c*(1/12)``, SE / SC the 12 edge / 8 corner neighbours summed
  sequentially in row-major offset order.  Chosen when every cell
  coefficient equals the first and it is > 0 (operators.py:172-176).
* table apply: 27 taps row-major (operators.py:229-239).
* d-linear P / R: axis 0, then 1, then 2, the reference's 1D DAGs.
* BoxMG P: c-points identity; edge points: 27-point rows lumped over the 9
  normal taps (row-major, sequential) -> the reference's closed-form 2x2;
  face points: rows lumped along the face normal (3 taps, sequential) -> the
  reference's 2D 4x4 solve; cell-interior points: the full rows -> 8x8
  solve.  Solves: LU with partial pivoting (first max |a|), multipliers by
  the reciprocal pivot, substitution by division (``lu_solve``; the CUDA
  kernel is the same sequence).
* Galerkin rows: the reference's loop order (operators.py:446-478) over
  125 fine offsets x 27 taps x 27 coarse neighbours.
* adaFACx R~: ``R( A1(x) * ((omega*3.0)/8.0) )`` with ``A1`` the unit
  constant operator (c = 1) and R the level's restriction (d-linear or
  BoxMG) -- the geometric fast path of operators.py:602-605, used for both
  flavours (mathematically omega R A1 diag(A1)^-1, operators.py:484-547).
* residual norm weight ``h^(d/2)`` per composite vertex (``(h^1.5 r)^2``
  summed); linf and the update counts as in 2D.

Layout: level l has ``n = 3**l`` cells per axis; vertex fields ``(n+1,)*3``,
cell fields ``(n,)*3``, C-ordered ``[i, j, k]`` with i along x; stencil
tables ``(N, N, N, 27)`` (tap ``(di+1)*9 + (dj+1)*3 + (dk+1)``); BoxMG P
``(Nc, Nc, Nc, 5, 5, 5)`` over fine offsets -2..2.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field
from itertools import product

import numpy as np

NONE, INTERIOR_DOF, DIRICHLET, HANGING, OVERLAPPED = 0, 1, 2, 3, 4
VARIANTS = ("additive", "additive-exp", "bpx", "afacc", "adafac-pi", "adafac-jac")

CORNERS = tuple((a0, a1, a2) for a2 in (0, 1) for a1 in (0, 1) for a0 in (0, 1))
OFFS27 = tuple(product((-1, 0, 1), repeat=3))
EDGE_OFFS = tuple(o for o in OFFS27 if sum(x != 0 for x in o) == 2)
CORNER_OFFS = tuple(o for o in OFFS27 if all(x != 0 for x in o))
K_D = 1.0 / 3.0
K_E = 1.0 / 12.0
C_D8 = 8.0 / 3.0
C_E6 = 1.0 / 6.0
C_C12 = 1.0 / 12.0


def element_matrix_unit() -> np.ndarray:
    """Trilinear stiffness of the unit cube, corner index a0 + 2 a1 + 4 a2 (for tests)."""
    M = np.array([[1.0 / 3.0, 1.0 / 6.0], [1.0 / 6.0, 1.0 / 3.0]])
    S = np.array([[1.0, -1.0], [-1.0, 1.0]])
    return (np.kron(M, np.kron(M, S)) + np.kron(M, np.kron(S, M))
            + np.kron(S, np.kron(M, M)))


def kmat(a: int, b: int) -> float:
    """Entry of K_unit as the kernels use it (0, K_D or -K_E)."""
    diff = sum(CORNERS[a][x] != CORNERS[b][x] for x in range(3))
    return K_D if diff == 0 else (0.0 if diff == 1 else -K_E)


def tap(o) -> int:
    return (o[0] + 1) * 9 + (o[1] + 1) * 3 + (o[2] + 1)


# -- shifted views -------------------------------------------------------------

def _sh(xp: np.ndarray, o, N: int, p: int = 1) -> np.ndarray:
    """x[v + o] for v in [0, N)^3 from a zero-padded copy (pad p)."""
    return xp[p + o[0]:p + o[0] + N, p + o[1]:p + o[1] + N, p + o[2]:p + o[2] + N]


def _cell_at(ep: np.ndarray, a, N: int) -> np.ndarray:
    """Coefficient of cell v - a for every vertex v (zero outside), ep padded by 1."""
    return ep[1 - a[0]:1 - a[0] + N, 1 - a[1]:1 - a[1] + N, 1 - a[2]:1 - a[2] + N]


def _seq_sum(terms):
    it = iter(terms)
    acc = next(it).copy()
    for t in it:
        acc = acc + t
    return acc


# -- operators -------------------------------------------------------------------

def apply_const(x: np.ndarray, c: float) -> np.ndarray:
    N = x.shape[0]
    xp = np.pad(x, 1)
    se = _seq_sum(_sh(xp, o, N) for o in EDGE_OFFS)
    sc = _seq_sum(_sh(xp, o, N) for o in CORNER_OFFS)
    m, e, k = c * C_D8, c * C_E6, c * C_C12
    return ((m * x) - (e * se)) - (k * sc)


def element_sums(x: np.ndarray, e: np.ndarray):
    """E (coefficient sum) and T (weighted far-corner sums) of the element apply."""
    N = x.shape[0]
    xp = np.pad(x, 1)
    ep = np.pad(e, 1)
    E = None
    T = None
    for a in CORNERS:
        s = tuple(1 - 2 * ai for ai in a)
        ec = _cell_at(ep, a, N)
        sc = ((_sh(xp, (s[0], s[1], 0), N) + _sh(xp, (s[0], 0, s[2]), N))
              + _sh(xp, (0, s[1], s[2]), N)) + _sh(xp, s, N)
        E = ec.copy() if E is None else E + ec
        T = ec * sc if T is None else T + ec * sc
    return E, T


def apply_element(x: np.ndarray, e: np.ndarray) -> np.ndarray:
    E, T = element_sums(x, e)
    return ((K_D * E) * x) - (K_E * T)


def element_diag(e: np.ndarray) -> np.ndarray:
    N = e.shape[0] + 1
    ep = np.pad(e, 1)
    E = _seq_sum(_cell_at(ep, a, N) for a in CORNERS)
    return K_D * E


def assemble_table(e: np.ndarray) -> np.ndarray:
    """Per-vertex 27-point rows from the adjacent element matrices, corner order a, b."""
    N = e.shape[0] + 1
    ep = np.pad(e, 1)
    t = np.zeros((N, N, N, 27))
    for ia, a in enumerate(CORNERS):
        ec = _cell_at(ep, a, N)
        for ib, b in enumerate(CORNERS):
            kab = kmat(ia, ib)
            if kab == 0.0:
                continue
            k = tap(tuple(b[x] - a[x] for x in range(3)))
            t[..., k] = t[..., k] + kab * ec
    return t


def apply_table(x: np.ndarray, t: np.ndarray) -> np.ndarray:
    N = x.shape[0]
    xp = np.pad(x, 1)
    out = np.zeros_like(x)
    for o in OFFS27:
        out = out + t[..., tap(o)] * _sh(xp, o, N)
    return out


class Op:
    """'const' / 'element' (per-cell coefficient e = eff*h) / 'table'."""

    def __init__(self, e: np.ndarray | None = None, table: np.ndarray | None = None):
        self.e, self.tbl = e, table
        self.kind, self.c = "table", None
        if table is None:
            first = float(e.flat[0])
            self.c = first if first > 0.0 and np.all(e == first) else None
            self.kind = "const" if self.c is not None else "element"
        self._diag = None

    def apply(self, x):
        if self.kind == "const":
            return apply_const(x, self.c)
        if self.kind == "element":
            return apply_element(x, self.e)
        return apply_table(x, self.tbl)

    def diag(self):
        if self._diag is None:
            self._diag = element_diag(self.e) if self.tbl is None else self.tbl[..., 13].copy()
        return self._diag

    def table(self):
        return assemble_table(self.e) if self.tbl is None else self.tbl


# -- d-linear transfers ----------------------------------------------------------

_W5 = np.array([1.0, 2.0, 3.0, 2.0, 1.0]) / 3.0


def _prolong_axis0(c: np.ndarray) -> np.ndarray:
    m = c.shape[0] - 1
    q, r = np.divmod(np.arange(3 * m + 1), 3)
    wl = (1.0 - r / 3.0).reshape((-1,) + (1,) * (c.ndim - 1))
    out = wl * c[q]
    out += (1.0 - wl) * c[np.minimum(q + 1, m)]
    return out


def _restrict_axis0(f: np.ndarray) -> np.ndarray:
    m = (f.shape[0] - 1) // 3
    out = np.zeros((m + 1,) + f.shape[1:])
    for k, off in enumerate(range(-2, 3)):
        lo = 1 if off < 0 else 0
        hi = m - 1 if off > 0 else m
        out[lo:hi + 1] += _W5[k] * f[3 * np.arange(lo, hi + 1) + off]
    return out


def _on_axis(fn, x, ax):
    return np.moveaxis(fn(np.moveaxis(x, ax, 0)), 0, ax)


def prolong_dlinear(c: np.ndarray) -> np.ndarray:
    """Axis 0, then 1, then 2 (operators.py:96-127 carried to 3D)."""
    for ax in range(3):
        c = _on_axis(_prolong_axis0, c, ax)
    return np.ascontiguousarray(c)


def restrict_dlinear(f: np.ndarray) -> np.ndarray:
    """Axis 0, then 1, then 2 (operators.py:111-132 carried to 3D)."""
    for ax in range(3):
        f = _on_axis(_restrict_axis0, f, ax)
    return np.ascontiguousarray(f)


def dlinear_p_table(nc: int) -> np.ndarray:
    """The d-linear weights in the BoxMG P layout: ((w_a * w_b) * w_c), w_o = max(0, 1 - |o|/3),
    zero where the fine offset leaves the grid (the throttled start, and tests)."""
    w = np.maximum(0.0, 1.0 - np.abs(np.arange(-2, 3)) / 3.0)
    w3 = (w[:, None, None] * w[None, :, None]) * w[None, None, :]
    p = np.broadcast_to(w3, (nc + 1,) * 3 + (5, 5, 5)).copy()
    idx = 3 * np.arange(nc + 1)
    for o in range(-2, 3):
        out = (idx + o < 0) | (idx + o > 3 * nc)
        p[out, :, :, o + 2] = 0.0
        p[:, out, :, :, o + 2] = 0.0
        p[:, :, out, :, :, o + 2] = 0.0
    return p


# -- BoxMG (operator-dependent) prolongation -------------------------------------

def lu_solve(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Batched A X = B by LU with partial pivoting (dgetf2 / dgetrs order).

    Pivot = first row of max |a| in the column; multipliers ``a * (1/pivot)``;
    forward substitution then back substitution by division.
    """
    A = A.copy()
    B = B.copy()
    m, n, _ = A.shape
    ar = np.arange(m)
    piv = np.zeros((m, n), dtype=np.int64)
    for k in range(n):
        p = k + np.argmax(np.abs(A[:, k:, k]), axis=1)
        piv[:, k] = p
        rk, rp_ = A[ar, k, :].copy(), A[ar, p, :].copy()
        A[ar, k, :] = rp_
        A[ar, p, :] = rk
        rp = 1.0 / A[:, k, k]
        for r in range(k + 1, n):
            A[:, r, k] = A[:, r, k] * rp
        for r in range(k + 1, n):
            for c in range(k + 1, n):
                A[:, r, c] = A[:, r, c] - A[:, r, k] * A[:, k, c]
    for k in range(n):
        p = piv[:, k]
        bk, bp = B[ar, k, :].copy(), B[ar, p, :].copy()
        B[ar, k, :] = bp
        B[ar, p, :] = bk
    for c in range(B.shape[2]):
        for k in range(n):
            for r in range(k + 1, n):
                B[:, r, c] = B[:, r, c] - B[:, k, c] * A[:, r, k]
        for k in range(n - 1, -1, -1):
            B[:, k, c] = B[:, k, c] / A[:, k, k]
            for r in range(k):
                B[:, r, c] = B[:, r, c] - B[:, k, c] * A[:, r, k]
    return B


def _pt(P: np.ndarray, W, o):
    """P[W, o] as an array over the coarse index arrays W (tuple of int arrays); 0 if |o|>2."""
    if any(abs(x) > 2 for x in o):
        return np.zeros(W[0].shape)
    return P[W[0], W[1], W[2], o[0] + 2, o[1] + 2, o[2] + 2]


def boxmg_p(tf: np.ndarray, nc: int) -> np.ndarray:
    """Operator-dependent P from the fine 27-point table tf (Nf^3 x 27), regular tree.

    3D analogue of boxmg_prolongation (operators.py:306-437).
    """
    Nc, Nf = nc + 1, 3 * nc + 1
    t6 = tf.reshape((Nf, Nf, Nf, 3, 3, 3))
    P = np.zeros((Nc, Nc, Nc, 5, 5, 5))
    P[..., 2, 2, 2] = 1.0
    # ---- edges along axis ax between W and W + e_ax: lump over the 9 normal taps
    for ax in range(3):
        others = [x for x in range(3) if x != ax]
        T = np.moveaxis(t6, 3 + ax, 3)  # (..., axial, o1, o2), o1 < o2 original order
        rng = [np.arange(Nc)] * 3
        rng[ax] = np.arange(nc)
        W = np.meshgrid(*rng, indexing="ij")
        W = tuple(w.ravel() for w in W)

        def lumped(step):
            f = [3 * W[x] for x in range(3)]
            f[ax] = f[ax] + step
            row = T[f[0], f[1], f[2]]  # (m, 3, 3, 3)
            return np.stack([_seq_sum(row[:, a, b, c] for b in range(3) for c in range(3))
                             for a in range(3)], axis=-1)

        c1, c2 = lumped(1), lumped(2)
        am1, a01, ap1 = c1[:, 0], c1[:, 1], c1[:, 2]
        am2, a02, ap2 = c2[:, 0], c2[:, 1], c2[:, 2]
        det = a01 * a02 - ap1 * am2
        scale = np.abs(a01 * a02) + np.abs(ap1 * am2)
        if (np.abs(det) <= 1e-14 * np.maximum(scale, 1e-300)).any():
            raise ArithmeticError("degenerate collapsed stencil in face-point solve")
        wl1 = (-am1) * a02 / det
        wl2 = am2 * am1 / det
        wh1 = ap1 * ap2 / det
        wh2 = a01 * (-ap2) / det
        Wh = list(W)
        Wh[ax] = W[ax] + 1
        for off, val, base in ((1, wl1, W), (2, wl2, W), (-2, wh1, Wh), (-1, wh2, Wh)):
            o = [2, 2, 2]
            o[ax] += off
            P[base[0], base[1], base[2], o[0], o[1], o[2]] = val
        del others
    # ---- faces with normal nx, in-plane axes p < q: lump along the normal, 2D 4x4 solve
    interior2 = ((1, 1), (2, 1), (1, 2), (2, 2))
    corner2 = ((0, 0), (3, 0), (0, 3), (3, 3))
    for nx in range(3):
        p_ax, q_ax = [x for x in range(3) if x != nx]
        rng = [np.arange(Nc)] * 3
        rng[p_ax] = np.arange(nc)
        rng[q_ax] = np.arange(nc)
        W = tuple(w.ravel() for w in np.meshgrid(*rng, indexing="ij"))
        m = W[0].size

        def vec(al, be):
            v = [0, 0, 0]
            v[p_ax], v[q_ax] = al, be
            return v

        def known(al, be):
            """(m, 4) weights of patch point (al, be) w.r.t. the 4 face corners, from P."""
            out = np.zeros((m, 4))
            for c, (cp, cq) in enumerate(corner2):
                cv = vec(cp // 3, cq // 3)
                Wc = tuple(W[x] + cv[x] for x in range(3))
                pv = vec(al, be)
                o = tuple(pv[x] - 3 * cv[x] for x in range(3))
                out[:, c] = _pt(P, Wc, o)
            return out

        A = np.zeros((m, 4, 4))
        R = np.zeros((m, 4, 4))
        for r, (fp, fq) in enumerate(interior2):
            fv = vec(fp, fq)
            f = [3 * W[x] + fv[x] for x in range(3)]
            row = t6[f[0], f[1], f[2]]  # (m, 3, 3, 3) taps by axis
            for da in (-1, 0, 1):
                for db in (-1, 0, 1):
                    terms = []
                    for dc in (-1, 0, 1):
                        tv = [0, 0, 0]
                        tv[p_ax], tv[q_ax], tv[nx] = da + 1, db + 1, dc + 1
                        terms.append(row[:, tv[0], tv[1], tv[2]])
                    coef = _seq_sum(terms)
                    tgt = (fp + da, fq + db)
                    if tgt in interior2:
                        A[:, r, interior2.index(tgt)] += coef
                    else:
                        R[:, r, :] -= coef[:, None] * known(*tgt)
        sol = lu_solve(A, R)
        for c, (cp, cq) in enumerate(corner2):
            cv = vec(cp // 3, cq // 3)
            Wc = tuple(W[x] + cv[x] for x in range(3))
            for r, (fp, fq) in enumerate(interior2):
                pv = vec(fp, fq)
                o = [pv[x] - 3 * cv[x] + 2 for x in range(3)]
                P[Wc[0], Wc[1], Wc[2], o[0], o[1], o[2]] = sol[:, r, c]
    # ---- cell interiors: 8x8 solve with the full 27-point rows
    interior3 = tuple((a, b, c) for c in (1, 2) for b in (1, 2) for a in (1, 2))
    C = tuple(w.ravel() for w in np.meshgrid(*([np.arange(nc)] * 3), indexing="ij"))
    m = C[0].size

    def known3(pt):
        out = np.zeros((m, 8))
        for ia, a in enumerate(CORNERS):
            Wc = tuple(C[x] + a[x] for x in range(3))
            o = tuple(pt[x] - 3 * a[x] for x in range(3))
            out[:, ia] = _pt(P, Wc, o)
        return out

    A = np.zeros((m, 8, 8))
    R = np.zeros((m, 8, 8))
    for r, pt in enumerate(interior3):
        f = [3 * C[x] + pt[x] for x in range(3)]
        row = tf[f[0], f[1], f[2]]  # (m, 27)
        for o in OFFS27:
            coef = row[:, tap(o)]
            tgt = tuple(pt[x] + o[x] for x in range(3))
            if tgt in interior3:
                A[:, r, interior3.index(tgt)] += coef
            else:
                R[:, r, :] -= coef[:, None] * known3(tgt)
    sol = lu_solve(A, R)
    for ia, a in enumerate(CORNERS):
        Wc = tuple(C[x] + a[x] for x in range(3))
        for r, pt in enumerate(interior3):
            o = [pt[x] - 3 * a[x] + 2 for x in range(3)]
            P[Wc[0], Wc[1], Wc[2], o[0], o[1], o[2]] = sol[:, r, ia]
    return P


def galerkin(fine_masked: np.ndarray, P: np.ndarray) -> np.ndarray:
    """Coarse 27-point rows of P^T A P, loop order of operators.py:446-478 in 3D."""
    Nc = P.shape[0]
    nc = Nc - 1
    Nf = 3 * nc + 1
    out = np.zeros((Nc, Nc, Nc, 27))
    pad = np.zeros((Nc + 2,) * 3 + (5, 5, 5))
    pad[1:-1, 1:-1, 1:-1] = P
    fpad = np.zeros((Nf + 4,) * 3 + (27,))
    fpad[2:-2, 2:-2, 2:-2] = fine_masked
    for o in product(range(-2, 3), repeat=3):
        r_w = P[..., o[0] + 2, o[1] + 2, o[2] + 2]
        if not np.any(r_w):
            continue
        sl = tuple(slice(2 + o[x], 2 + o[x] + 3 * nc + 1, 3) for x in range(3))
        arow = fpad[sl]
        for s in OFFS27:
            acoef = arow[..., tap(s)]
            t = tuple(o[x] + s[x] for x in range(3))
            for dw in OFFS27:
                pw_o = tuple(t[x] - 3 * dw[x] for x in range(3))
                if any(abs(v) > 2 for v in pw_o):
                    continue
                p_w = pad[1 + dw[0]:Nc + 1 + dw[0], 1 + dw[1]:Nc + 1 + dw[1], 1 + dw[2]:Nc + 1 + dw[2],
                          pw_o[0] + 2, pw_o[1] + 2, pw_o[2] + 2]
                k = tap(dw)
                out[..., k] = out[..., k] + (r_w * acoef) * p_w
    return out


class Transfer:
    """Transfers between coarse level l (nc = 3**l) and l + 1."""

    def __init__(self, nc: int, P: np.ndarray | None, omega: float | None):
        self.nc, self.p, self.omega = nc, P, omega

    def prolong(self, c: np.ndarray) -> np.ndarray:
        if self.p is None:
            return prolong_dlinear(c)
        nc, Nf = self.nc, 3 * self.nc + 1
        fine = np.zeros((Nf,) * 3)
        idx = np.arange(nc + 1)
        for o in product(range(-2, 3), repeat=3):
            w = self.p[..., o[0] + 2, o[1] + 2, o[2] + 2]
            if not np.any(w):
                continue
            sel = []
            for x in range(3):
                ok = (3 * idx + o[x] >= 0) & (3 * idx + o[x] <= Nf - 1)
                sel.append(idx[ok])
            lo = [s[0] for s in sel]
            hi = [s[-1] for s in sel]
            fsl = tuple(slice(3 * lo[x] + o[x], 3 * hi[x] + o[x] + 1, 3) for x in range(3))
            csl = tuple(slice(lo[x], hi[x] + 1) for x in range(3))
            fine[fsl] += (w * c)[csl]
        return fine

    def _gather(self, f: np.ndarray, o) -> np.ndarray:
        nc = self.nc
        fp = np.pad(f, 2)
        return fp[tuple(slice(2 + o[x], 2 + o[x] + 3 * nc + 1, 3) for x in range(3))]

    def restrict(self, f: np.ndarray) -> np.ndarray:
        if self.p is None:
            return restrict_dlinear(f)
        out = np.zeros((self.nc + 1,) * 3)
        for o in product(range(-2, 3), repeat=3):
            w = self.p[..., o[0] + 2, o[1] + 2, o[2] + 2]
            if not np.any(w):
                continue
            out += w * self._gather(f, o)
        return out

    def restrict_smoothed(self, f: np.ndarray) -> np.ndarray:
        s = apply_const(f, 1.0)
        s *= self.omega * 3.0 / 8.0
        return self.restrict(s)


# -- mesh ---------------------------------------------------------------------------

class Tree:
    """Regular 3D tripartitioned spacetree: levels 0..depth, all cells of levels < depth refined."""

    def __init__(self, levels: int, lmin: int = 1):
        if levels < 1:
            raise ValueError("need at least one refined level to obtain DoFs")
        self.lmin, self.lmax = lmin, levels
        self.u = [np.zeros((3**l + 1,) * 3) for l in range(levels + 1)]
        self.eps = [np.ones((3**l,) * 3) for l in range(levels + 1)]

    @property
    def depth(self) -> int:
        return self.lmax

    def kinds(self, l: int) -> np.ndarray:
        N = 3**l + 1
        k = np.full((N, N, N), DIRICHLET, dtype=np.int8)
        k[1:-1, 1:-1, 1:-1] = OVERLAPPED if l < self.depth else INTERIOR_DOF
        return k


def child_mean(e: np.ndarray) -> np.ndarray:
    """Mean of the 27 children: sequential sum in row-major child order, / 27."""
    n = e.shape[0] // 3
    r = e.reshape(n, 3, n, 3, n, 3)
    return _seq_sum(r[:, a, :, b, :, c] for a in range(3) for b in range(3) for c in range(3)) / 27.0


# -- engine ----------------------------------------------------------------------------

@dataclass
class Config:
    variant: str = "adafac-jac"
    flavor: str = "geometric"
    omega: float = 0.6
    omega_tilde: float | None = None
    omega_hat: float = 0.7
    damping_scale: float = 1.0
    # BoxMG only: start from d-linear P and rediscretised coarse operators and
    # replace them by BoxMG P / Galerkin rows one level per cycle, finest first
    # (the paper's throttled operator propagation; the
    # reference builds every level eagerly, solvers.py:227-250)
    throttled: bool = False

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
    """ReferenceEngine (solvers.py:129-492) carried to 3D regular trees."""

    def __init__(self, tree: Tree, cfg: Config):
        if cfg.variant not in VARIANTS or cfg.flavor not in ("geometric", "boxmg"):
            raise ValueError("bad config")
        self.tree, self.cfg = tree, cfg
        self.rhs: dict[int, np.ndarray] = {}
        self.rebuild()

    def rebuild(self) -> None:
        t, cfg = self.tree, self.cfg
        self.ltop = top = t.depth
        l0 = t.lmin
        self.eff = {top: t.eps[top].copy()}
        for l in range(top - 1, l0 - 1, -1):
            self.eff[l] = child_mean(self.eff[l + 1])
        self.coef = {l: self.eff[l] * (3.0 ** -l) for l in range(l0, top + 1)}
        self.masks, self.ops, self.tr, self.hw = {}, {}, {}, {}
        for l in range(l0, top + 1):
            k = t.kinds(l)
            dof = (k == INTERIOR_DOF) | (k == OVERLAPPED)
            self.masks[l] = dict(kinds=k, dof=dof, composite=k == INTERIOR_DOF,
                                 exists=k != NONE, overlapped=k == OVERLAPPED, rho_src=dof)
            self.hw[l] = 3.0 ** (-1.5 * l)
        self.ptab = {}
        if cfg.flavor == "geometric":
            for l in range(l0, top + 1):
                self.ops[l] = Op(self.coef[l])
            for l in range(l0, top):
                self.tr[l] = Transfer(3**l, None, cfg.omega)
        else:
            self.ops[top] = Op(self.coef[top])
            self.thr_next = l0 - 1
            if cfg.throttled:
                for l in range(top - 1, l0 - 1, -1):
                    self.ops[l] = Op(table=assemble_table(self.coef[l]))
                    self.tr[l] = Transfer(3**l, dlinear_p_table(3**l), cfg.omega)
                self.thr_next = top - 1
            else:
                for l in range(top - 1, l0 - 1, -1):
                    self._build_boxmg_level(l)

    def _build_boxmg_level(self, l: int) -> None:
        """BoxMG P and Galerkin rows of level l from level l+1's operator (solvers.py:227-250)."""
        raw = self.ops[l + 1].table()
        P = boxmg_p(raw, 3**l)
        masked = raw * self.masks[l + 1]["dof"][..., None]
        rap = galerkin(masked, P)
        tbl = assemble_table(self.coef[l])
        ov = self.masks[l]["overlapped"]
        tbl[ov] = rap[ov]
        self.ops[l] = Op(table=tbl)
        self.tr[l] = Transfer(3**l, P, self.cfg.omega)

    def update_fas_state(self) -> None:
        t = self.tree
        for l in range(self.ltop - 1, t.lmin - 1, -1):
            fk = self.masks[l + 1]["kinds"][::3, ::3, ::3]
            take = (fk == INTERIOR_DOF) | (fk == OVERLAPPED)
            t.u[l][take] = t.u[l + 1][::3, ::3, ::3][take]

    def _rhs(self, l: int) -> np.ndarray:
        r = self.rhs.get(l)
        return np.zeros_like(self.tree.u[l]) if r is None else r

    def _w(self, l: int) -> float:
        if self.cfg.variant == "additive-exp":
            return self.cfg.omega_hat ** (self.ltop - l)
        return self.cfg.omega

    def _stats_add(self, st: Stats, l: int, r: np.ndarray) -> None:
        comp = self.masks[l]["composite"]
        if comp.any():
            rr = r[comp]
            st.l2h += float(((self.hw[l] * rr) ** 2).sum())
            st.linf = max(st.linf, float(np.abs(rr).max()))
            st.dofs += int(comp.sum())
        st.level_dofs[l] = int(self.masks[l]["dof"].sum())

    def count_updates(self) -> int:
        l0, l1, v = self.tree.lmin, self.ltop, self.cfg.variant
        dof = {l: int(self.masks[l]["dof"].sum()) for l in range(l0, l1 + 1)}
        total = sum(dof.values())
        if v == "adafac-jac":
            total += sum(dof[l] for l in range(l0, l1))
        elif v == "adafac-pi":
            total += sum(dof[l] for l in range(l0 + 1, l1 + 1))
        return total

    def _bpart(self, l: int, au: np.ndarray) -> np.ndarray:
        # regular tree: every refined-region vertex that carries an equation is overlapped
        return np.where(self.masks[l]["overlapped"], au, 0.0)

    def advance(self) -> Stats:
        """One additive cycle; stats of the starting iterate (solvers.py:334-399)."""
        if self.cfg.flavor == "boxmg" and self.thr_next >= self.tree.lmin:
            self._build_boxmg_level(self.thr_next)  # throttled: one more level per cycle
            self.thr_next -= 1
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
                    src[::3, ::3, ::3] = 0.0
                b[l - 1] = self.tr[l - 1].restrict(src)
                b[l - 1] += self._rhs(l - 1)
            rho_below = rdof
        if cfg.variant == "adafac-pi":
            for l in range(l0 + 1, l1 + 1):
                inj = np.zeros_like(t.u[l - 1])
                fk = self.masks[l]["kinds"][::3, ::3, ::3]
                take = (fk == INTERIOR_DOF) | (fk == OVERLAPPED)
                inj[take] = d[l][::3, ::3, ::3][take]
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

    def residual_stats(self) -> Stats:
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
                    src[::3, ::3, ::3] = 0.0
                b[l - 1] = self.tr[l - 1].restrict(src) + self._rhs(l - 1)
        st.l2h = float(np.sqrt(st.l2h))
        return st
