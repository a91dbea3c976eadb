"""Pin the 3D CPU oracle (oracle/mg3d.py).

The reference is 2D only, so 3D parity is *unpinned by the reference*; these
tests pin the restatement by independent FE assembly and by the invariants the
reference's own tests check in 2D:

* trilinear stiffness from Gauss quadrature; operator apply / diagonal /
  tables equal a dense FE assembly (tests/test_discretization.py:19-47,
  tests/test_oracle.py:95-117 in 2D);
* d-linear and BoxMG restriction are P^T (tests/test_operators.py:64-72);
* BoxMG P equals trilinear for constant eps, reproduces constants, unit
  c-point rows (tests/test_operators.py:113-154);
* Galerkin rows equal P^T A P (tests/test_oracle.py:95-117);
* the exact discrete solution is a fixed point of every variant
  (tests/test_solvers.py:137-159); adaFACx with damping_scale 0 equals
  additive bit for bit (tests/test_solvers.py:225-234); geometric equals
  BoxMG on Poisson (tests/test_solvers.py:237-246); update counts
  (tests/test_solvers.py:249-269).
"""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import mg3d as m

RNG = np.random.default_rng(1234)


def gauss_stiffness():
    """Unit-cube trilinear stiffness by 2-point Gauss quadrature (independent of kron)."""
    g = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
    K = np.zeros((8, 8))
    for x in g:
        for y in g:
            for z in g:
                grads = []
                for (a0, a1, a2) in m.CORNERS:
                    fx = (x if a0 else 1 - x, 1.0 if a0 else -1.0)
                    fy = (y if a1 else 1 - y, 1.0 if a1 else -1.0)
                    fz = (z if a2 else 1 - z, 1.0 if a2 else -1.0)
                    grads.append([fx[1] * fy[0] * fz[0], fx[0] * fy[1] * fz[0], fx[0] * fy[0] * fz[1]])
                gr = np.array(grads)
                K += 0.125 * gr @ gr.T
    return K


def dense_fe(e):
    n = e.shape[0]
    N = n + 1
    K = gauss_stiffness()
    rows, cols, vals = [], [], []
    idx = lambda i, j, k: (i * N + j) * N + k  # noqa: E731
    for ci in range(n):
        for cj in range(n):
            for ck in range(n):
                vs = [idx(ci + a0, cj + a1, ck + a2) for (a0, a1, a2) in m.CORNERS]
                for a in range(8):
                    for b in range(8):
                        rows.append(vs[a])
                        cols.append(vs[b])
                        vals.append(e[ci, cj, ck] * K[a, b])
    return sp.csr_matrix((vals, (rows, cols)), shape=(N**3, N**3))


def table_matrix(t):
    N = t.shape[0]
    rows, cols, vals = [], [], []
    for v in range(N**3):
        i, j, k = np.unravel_index(v, (N,) * 3)
        for o in m.OFFS27:
            ii, jj, kk = i + o[0], j + o[1], k + o[2]
            if 0 <= ii < N and 0 <= jj < N and 0 <= kk < N:
                rows.append(v)
                cols.append((ii * N + jj) * N + kk)
                vals.append(t[i, j, k, m.tap(o)])
    return sp.csr_matrix((vals, (rows, cols)), shape=(N**3, N**3))


def prolong_matrix(tr, nc):
    Nc = nc + 1
    cols = []
    for k in range(Nc**3):
        ek = np.zeros(Nc**3)
        ek[k] = 1.0
        cols.append(tr.prolong(ek.reshape((Nc,) * 3)).ravel())
    return np.stack(cols, axis=1)


def test_element_matrix_is_trilinear_stiffness():
    np.testing.assert_allclose(m.element_matrix_unit(), gauss_stiffness(), atol=1e-15)
    K = gauss_stiffness()
    for a in range(8):
        for b in range(8):
            assert abs(K[a, b] - m.kmat(a, b)) < 1e-15


@pytest.mark.parametrize("n", [3, 9])
def test_operator_apply_diag_table_equal_fe_assembly(n):
    e = 10.0 ** RNG.uniform(-2, 2, (n,) * 3)
    N = n + 1
    A = dense_fe(e)
    x = RNG.standard_normal((N,) * 3)
    want = (A @ x.ravel()).reshape((N,) * 3)
    sc = np.abs(want).max()
    assert np.abs(m.apply_element(x, e) - want).max() <= 1e-14 * sc
    t = m.assemble_table(e)
    assert np.abs(m.apply_table(x, t) - want).max() <= 1e-14 * sc
    assert np.abs(table_matrix(t).toarray() - A.toarray()).max() <= 1e-14 * np.abs(e).max()
    np.testing.assert_allclose(m.element_diag(e), A.diagonal().reshape((N,) * 3), rtol=1e-14)
    # constant fast path equals the assembled operator on interior vertices
    c = 0.37
    Ac = dense_fe(np.full((n,) * 3, c))
    wc = (Ac @ x.ravel()).reshape((N,) * 3)
    inner = (slice(1, -1),) * 3
    np.testing.assert_allclose(m.apply_const(x, c)[inner], wc[inner], rtol=0, atol=1e-14 * np.abs(wc).max())


def test_dlinear_restriction_is_transpose():
    nc = 3
    tr = m.Transfer(nc, None, 0.6)
    Pm = prolong_matrix(tr, nc)
    f = RNG.standard_normal((3 * nc + 1,) * 3)
    np.testing.assert_allclose(tr.restrict(f).ravel(), Pm.T @ f.ravel(), rtol=0, atol=1e-13)
    np.testing.assert_allclose(m.Transfer(nc, m.dlinear_p_table(nc), 0.6).prolong(
        np.arange(64.0).reshape(4, 4, 4)), tr.prolong(np.arange(64.0).reshape(4, 4, 4)), atol=1e-13)


def test_boxmg_properties():
    nc = 3
    tf = m.assemble_table(np.full((9, 9, 9), 1.0 / 9.0))
    np.testing.assert_allclose(m.boxmg_p(tf, nc), m.dlinear_p_table(nc), atol=1e-14)
    e = 10.0 ** RNG.uniform(-2, 2, (9, 9, 9))
    P = m.boxmg_p(m.assemble_table(e), nc)
    assert np.all(P[..., 2, 2, 2] == 1.0)
    tr = m.Transfer(nc, P, 0.6)
    np.testing.assert_allclose(tr.prolong(np.ones((4, 4, 4))), 1.0, atol=1e-13)
    # scale invariance
    P2 = m.boxmg_p(m.assemble_table(e * 7.0), nc)
    np.testing.assert_allclose(P2, P, atol=1e-13)
    Pm = prolong_matrix(tr, nc)
    f = RNG.standard_normal((10,) * 3)
    np.testing.assert_allclose(tr.restrict(f).ravel(), Pm.T @ f.ravel(), atol=1e-13)


def test_galerkin_equals_ptap():
    nc = 3
    e = 10.0 ** RNG.uniform(-2, 2, (9, 9, 9))
    tf = m.assemble_table(e)
    P = m.boxmg_p(tf, nc)
    dof = np.zeros((10,) * 3, bool)
    dof[1:-1, 1:-1, 1:-1] = True
    masked = tf * dof[..., None]
    Pm = prolong_matrix(m.Transfer(nc, P, 0.6), nc)
    G = Pm.T @ table_matrix(masked).toarray() @ Pm
    rap = m.galerkin(masked, P)
    np.testing.assert_allclose(table_matrix(rap).toarray(), G, rtol=0, atol=1e-14 * np.abs(G).max())
    # unit coefficient: Galerkin of trilinear P equals rediscretisation on interior rows
    t1 = m.assemble_table(np.full((9, 9, 9), 1.0))
    r1 = m.galerkin(t1 * dof[..., None], m.dlinear_p_table(nc))
    t3 = m.assemble_table(np.full((3, 3, 3), 3.0))
    np.testing.assert_allclose(r1[1:-1, 1:-1, 1:-1], t3[1:-1, 1:-1, 1:-1], atol=1e-13)


def make(L, flavor, variant="adafac-jac", blocks=False, seed=0, ds=1.0, throttled=False):
    t = m.Tree(L)
    rng = np.random.default_rng(seed)
    n = 3**L
    if blocks:
        blk = 3 ** max(L - 3, 0)
        b = 10.0 ** rng.uniform(-2, 2, (n // blk,) * 3)
        t.eps[L] = np.kron(b, np.ones((blk,) * 3))
    eng = m.Engine(t, m.Config(variant=variant, flavor=flavor, damping_scale=ds, throttled=throttled))
    f = rng.uniform(-1, 1, (n - 1,) * 3)
    rhs = np.zeros((n + 1,) * 3)
    rhs[1:-1, 1:-1, 1:-1] = (3.0 ** -L) ** 3 * f
    eng.rhs[L] = rhs
    return t, eng


@pytest.mark.parametrize("variant", m.VARIANTS)
@pytest.mark.parametrize("flavor", ["geometric", "boxmg"])
def test_exact_solution_is_fixed_point(variant, flavor):
    L = 2
    t, eng = make(L, flavor, variant, blocks=True)
    N = 3**L + 1
    A = table_matrix(eng.ops[L].table()).tocsr()
    inner = np.zeros((N,) * 3, bool)
    inner[1:-1, 1:-1, 1:-1] = True
    ii = np.flatnonzero(inner.ravel())
    sol = np.zeros(N**3)
    sol[ii] = spla.spsolve(A[ii][:, ii].tocsc(), eng.rhs[L].ravel()[ii])
    t.u[L][...] = sol.reshape((N,) * 3)
    eng.update_fas_state()
    before = [u.copy() for u in t.u]
    st = eng.advance()
    assert st.l2h <= 1e-12 * np.abs(eng.rhs[L]).max()
    for l in range(1, L + 1):
        np.testing.assert_allclose(t.u[l], before[l], rtol=0, atol=1e-13)


def test_adafac_ds0_equals_additive_bitwise():
    t1, e1 = make(3, "boxmg", "adafac-jac", blocks=True, ds=0.0)
    t2, e2 = make(3, "boxmg", "additive", blocks=True)
    for _ in range(3):
        a, b = e1.advance(), e2.advance()
        assert a.l2h == b.l2h
    assert np.array_equal(t1.u[3], t2.u[3])


def test_geometric_equals_boxmg_on_poisson():
    t1, e1 = make(3, "geometric", "adafac-jac")
    t2, e2 = make(3, "boxmg", "adafac-jac")
    h1 = [e1.advance().l2h for _ in range(5)]
    h2 = [e2.advance().l2h for _ in range(5)]
    np.testing.assert_allclose(h1, h2, rtol=1e-11)


@pytest.mark.parametrize("flavor", ["geometric", "boxmg"])
def test_cycle_converges_and_counts(flavor):
    t, eng = make(3, flavor, "adafac-jac", blocks=flavor == "boxmg")
    h = [eng.advance() for _ in range(12)]
    assert h[-1].l2h < 0.1 * h[0].l2h
    dofs = {l: (3**l - 1) ** 3 for l in range(1, 4)}
    assert h[0].dofs == dofs[3]
    assert h[0].updates == sum(dofs.values()) + dofs[1] + dofs[2]


def test_throttled_setup_reaches_the_eager_operators():
    """Throttled BoxMG: cycle 1 already uses BoxMG on the level
    below the top; after top - lmin cycles every P and Galerkin table equals the
    eager build bitwise and the two runs converge alike."""
    t1, e1 = make(3, "boxmg", "adafac-jac", blocks=True)
    t2, e2 = make(3, "boxmg", "adafac-jac", blocks=True, throttled=True)
    # before any cycle: d-linear P and rediscretised rows on every coarse level
    for l in (1, 2):
        assert np.array_equal(e2.tr[l].p, m.dlinear_p_table(3**l))
        assert np.array_equal(e2.ops[l].tbl, m.assemble_table(e2.coef[l]))
    h1 = [e1.advance().l2h for _ in range(12)]
    h2 = [e2.advance().l2h for _ in range(12)]
    assert h2[0] == h1[0]  # stats of the starting iterate
    assert h2[1] != h1[1]  # level 1 is still d-linear in cycle 1
    for l in (1, 2):
        assert np.array_equal(e1.tr[l].p, e2.tr[l].p)
        assert np.array_equal(e1.ops[l].tbl, e2.ops[l].tbl)
    assert h2[-1] < 0.1 * h2[0]
    np.testing.assert_allclose(h2[-1], h1[-1], rtol=0.5)


def test_dlinear_p_table_equals_dlinear_prolongation():
    """The d-linear weights in the P layout prolong like the separable transfer."""
    nc = 3
    rng = np.random.default_rng(3)
    xc = np.zeros((nc + 1,) * 3)
    xc[1:-1, 1:-1, 1:-1] = rng.standard_normal((nc - 1,) * 3)
    a = m.Transfer(nc, None, 0.6).prolong(xc)
    b = m.Transfer(nc, m.dlinear_p_table(nc), 0.6).prolong(xc)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-14)
