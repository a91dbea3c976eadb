"""GPU parity of the 3D engine (libtmg.so through GpuEngine) against the 3D oracle.

There is no 3D reference (treemg is 2D only); the oracle ``oracle/mg3d.py``
defines the fp64 expression DAG of every 3D operation and the kernels evaluate
the same algorithm with FMA contraction (the 3D translation unit is built with
``--fmad=true``; there is no 3D reference to pin rounding to).  The bar is the
north star's: per-cycle residual 2-norms (and max norms) and the final ``u``
on every level within relative 1e-10 (``RTOL``; ``u`` normwise per level), P
and Galerkin tables within 1e-12.  Depth 4 and depth 5 -- including config
5's 27-cell coefficient blocks, where the weight dictionaries of the
config-5 bench path engage -- are checked against committed fixtures
(tests/golden3d, made by tests/golden3d/make_golden3d.py from the oracle):
per-cycle history, per-level norms and a strided sample of the final iterate.
"""

import json
import os

import numpy as np
import pytest

from oracle import mg3d
from paper_1903_10367_b200 import GpuEngine, SolverConfig, workloads

pytestmark = pytest.mark.gpu
RTOL = 1e-10  # BASELINE.json north star: residual history and final u within relative 1e-10

HERE = os.path.dirname(os.path.abspath(__file__))


def oracle_run(wl, n, variant=None, flavor=None, **kw):
    t = mg3d.Tree(wl.tree.depth, wl.tree.lmin)
    t.eps[wl.tree.depth] = wl.tree.eps[wl.tree.depth].copy()
    for l in range(len(t.u)):
        t.u[l] = wl.tree.u[l].copy()
    cfg = mg3d.Config(variant=variant or wl.variant, flavor=flavor or wl.flavor, **kw)
    e = mg3d.Engine(t, cfg)
    e.rhs.update({l: b.copy() for l, b in wl.rhs.items()})
    hist = [e.advance() for _ in range(n)]
    return t, e, hist


def gpu_run(wl, n, variant=None, flavor=None, **kw):
    cfg = SolverConfig(variant=variant or wl.variant, flavor=flavor or wl.flavor, **kw)
    eng = GpuEngine(wl.tree, cfg, sync="lazy")
    eng.rhs.update(wl.rhs)
    hist = eng.advance_many(n)
    eng.pull()
    return eng, hist


def close_u(got, want, rtol=RTOL, what="u"):
    """Normwise relative bound: max |got - want| <= rtol * max |want|."""
    scale = max(float(np.abs(want).max()), 1e-300)
    err = float(np.abs(got - want).max())
    assert err <= rtol * scale, f"{what}: max abs diff {err:.3e} > {rtol:g} x {scale:.3e}"


def check(wl, eng, hist, t, e, ohist):
    np.testing.assert_allclose([s.l2h for s in hist], [s.l2h for s in ohist], rtol=RTOL, atol=0)
    np.testing.assert_allclose([s.linf for s in hist], [s.linf for s in ohist], rtol=RTOL, atol=0)
    assert [s.dofs for s in hist] == [s.dofs for s in ohist]
    assert [s.updates for s in hist] == [s.updates for s in ohist]
    for l in range(wl.tree.lmin, wl.tree.depth + 1):
        close_u(wl.tree.u[l], t.u[l], what=f"u level {l}")


VARIANTS = ["additive", "additive-exp", "bpx", "afacc", "adafac-pi", "adafac-jac"]


@pytest.mark.parametrize("flavor", ["geometric", "boxmg"])
@pytest.mark.parametrize("variant", VARIANTS)
def test_3d_small_all_variants(variant, flavor):
    wl = workloads.config5(levels=2, block=3) if flavor == "boxmg" else workloads.config3(levels=2)
    t, e, oh = oracle_run(wl, 6, variant, flavor)
    eng, h = gpu_run(wl, 6, variant, flavor)
    check(wl, eng, h, t, e, oh)


@pytest.mark.parametrize("name", ["config3-small", "config5-small"])
def test_3d_level3(name):
    wl = workloads.by_name(name)
    t, e, oh = oracle_run(wl, 8)
    eng, h = gpu_run(wl, 8)
    check(wl, eng, h, t, e, oh)
    rs = eng.residual_stats()
    ors = e.residual_stats()
    np.testing.assert_allclose([rs.l2h, rs.linf], [ors.l2h, ors.linf], rtol=RTOL)


def test_3d_boxmg_tables():
    wl = workloads.config5(levels=3)
    t, e, _ = oracle_run(wl, 0)
    eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor))
    for l in range(wl.tree.lmin, wl.tree.depth):
        close_u(eng.transfers[l].p_table, e.tr[l].p, 1e-12, f"P level {l}")
        got = eng.ops[l].table().reshape(e.ops[l].tbl.shape)
        close_u(got, e.ops[l].tbl, 1e-12, f"A level {l}")
    for l in range(wl.tree.lmin, wl.tree.depth + 1):
        close_u(eng.eff_eps(l), e.eff[l], 1e-14, f"eff level {l}")


def test_3d_ds0_equals_additive_and_kinds():
    wl = workloads.config5(levels=3)
    e1, h1 = gpu_run(wl, 4, "adafac-jac", damping_scale=0.0)
    wl2 = workloads.config5(levels=3)
    e2, h2 = gpu_run(wl2, 4, "additive")
    np.testing.assert_allclose([s.l2h for s in h1], [s.l2h for s in h2], rtol=1e-13)
    close_u(wl.tree.u[3], wl2.tree.u[3], 1e-13)
    for l in (1, 2, 3):
        assert np.array_equal(e1.kinds(l), wl.tree.vertex_kinds(l))


FIXTURES = sorted(f[:-4] for f in os.listdir(os.path.join(HERE, "golden3d")) if f.endswith(".npz"))


@pytest.mark.parametrize("name", FIXTURES)
def test_3d_fixture_history_and_iterate(name):
    """Default engine vs the oracle's committed run (history, per-level norms, strided u sample)."""
    z = np.load(os.path.join(HERE, "golden3d", name + ".npz"))
    meta = json.loads(str(z["meta"]))
    wl = workloads.by_name(meta["workload"])
    eng, h = gpu_run(wl, meta["cycles"])
    if name == "config5-L5b27":  # the config-5 bench path: weight dictionaries engaged
        st = eng.weight_storage(wl.tree.depth - 1)
        assert 0 < st["p_distinct"] <= st["p_rows"] // 4, st
        assert 0 < st["pc_distinct"] <= st["pc_rows"] // 4, st
        assert 0 < st["galerkin_stored"] <= st["galerkin_rows"] // 2, st  # run-length Galerkin rows
    if name == "random-L5":  # per-cell coefficients: the dense weight streams
        st = eng.weight_storage(wl.tree.depth - 1)
        assert st["p_distinct"] == 0 and st["pc_distinct"] == 0 and st["galerkin_stored"] == 0, st
    np.testing.assert_allclose([s.l2h for s in h], z["l2h"], rtol=RTOL)
    np.testing.assert_allclose([s.linf for s in h], z["linf"], rtol=RTOL)
    s = meta["stride"]
    for l in range(wl.tree.lmin, wl.tree.depth + 1):
        u = wl.tree.u[l]
        o = l % s
        close_u(u[o::s, o::s, o::s], z[f"sample_{l}"], what=f"u sample level {l}")
        nrm = z[f"norms_{l}"]
        np.testing.assert_allclose([(u * u).sum(), np.abs(u).max()], nrm[1:], rtol=RTOL)
        assert abs(u.sum() - nrm[0]) <= RTOL * np.abs(u).sum()


@pytest.mark.parametrize("name,variant", [("config5-small", "adafac-jac"), ("config5-L4", "adafac-jac"),
                                          ("config5-L4", "additive"), ("config5-L4", "bpx")])
def test_3d_throttled_setup(name, variant):
    """Throttled BoxMG setup (one level per cycle, finest first) matches the oracle;
    once every level is upgraded the P and Galerkin tables equal the eager build's."""
    wl = workloads.by_name(name)
    top, lmin = wl.tree.depth, wl.tree.lmin
    n = top - lmin + 2
    t, e, oh = oracle_run(wl, n, variant, throttled=True)
    eng, h = gpu_run(wl, n, variant, throttled=True)
    check(wl, eng, h, t, e, oh)
    _, e_eager, _ = oracle_run(workloads.by_name(name), 0, variant)
    for l in range(lmin, top):
        close_u(eng.transfers[l].p_table, e_eager.tr[l].p, 1e-12, f"P level {l}")
        got = eng.ops[l].table().reshape(e_eager.ops[l].tbl.shape)
        close_u(got, e_eager.ops[l].tbl, 1e-12, f"A level {l}")


def test_3d_throttled_rebuild_restarts():
    wl = workloads.by_name("config5-small")
    eng, h1 = gpu_run(wl, 3, throttled=True)
    wl2 = workloads.by_name("config5-small")
    eng2, _ = gpu_run(wl2, 0, throttled=True)
    for l in range(len(wl2.tree.u)):
        eng.tree.u[l][...] = wl2.tree.u[l]
    eng.rebuild()
    h2 = eng.advance_many(3)
    np.testing.assert_allclose([s.l2h for s in h2], [s.l2h for s in h1], rtol=1e-13)


def test_3d_rebuild_after_shard_is_unsharded():
    """tmg3_rebuild on a sharded handle drops the shard state (its buffers were freed)."""
    import ctypes as C

    from paper_1903_10367_b200 import _abi
    wl = workloads.config5(levels=3)
    eng, h1 = gpu_run(wl, 2)
    L = _abi.lib()
    lo = (C.c_int32 * 4)(0, 0, 0, 0)
    hi = (C.c_int32 * 4)(0, 0, 0, 28)
    _abi.check(L.tmg3_shard(eng._h, 3, lo, hi))
    wl2 = workloads.config5(levels=3)
    for l in range(len(wl2.tree.u)):
        eng.tree.u[l][...] = wl2.tree.u[l]
    eng.rebuild()
    with pytest.raises(ValueError, match="not sharded"):
        _abi.check(L.tmg3_phase(eng._h, _abi.PH_DOWN, 3))
    with pytest.raises(ValueError, match="DOWN and UP only"):
        _abi.check(L.tmg3_phase_range(eng._h, _abi.PH_REDUCE, 3, 1, 5, 1, 1))
    h2 = eng.advance_many(2)
    np.testing.assert_allclose([s.l2h for s in h2], [s.l2h for s in h1], rtol=1e-13)


def test_3d_error_paths_raise_like_the_reference():
    import ctypes as C

    from paper_1903_10367_b200 import _abi, sharding
    wl = workloads.config5(levels=2, block=3)
    with pytest.raises(ValueError):
        GpuEngine(wl.tree, SolverConfig(variant="multiplicative-v10", flavor="boxmg"))
    with pytest.raises(ValueError, match="throttled"):
        GpuEngine(wl.tree, SolverConfig(variant="adafac-jac", flavor="geometric", throttled=True))
    with pytest.raises(ValueError, match="rtilde_true_operator"):
        GpuEngine(wl.tree, SolverConfig(variant="adafac-jac", flavor="boxmg", rtilde_true_operator=True))
    wl = workloads.config5(levels=3)
    eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
    L = _abi.lib()
    with pytest.raises(ValueError, match="not sharded"):
        _abi.check(L.tmg3_phase(eng._h, _abi.PH_DOWN, 3))
    lo = (C.c_int32 * 4)(0, 0, 0, 0)
    hi = (C.c_int32 * 4)(0, 0, 0, 99)  # beyond the level
    with pytest.raises(ValueError, match="plane range"):
        _abi.check(L.tmg3_shard(eng._h, 2, lo, hi))
    with pytest.raises(ValueError):
        _abi.check(L.tmg_get_u(eng._h, 9, None))
    with pytest.raises(ValueError):
        sharding.plan(2, 8)  # too shallow for 8 ranks


@pytest.mark.parametrize("variant", ["adafac-jac", "additive", "afacc"])
@pytest.mark.parametrize("wname", ["config5-L5", "random-L5"])
def test_3d_weight_dictionary_equals_dense(variant, wname, monkeypatch):
    """Level ltop-1's BoxMG weights as bitwise-verified row dictionaries (k3_smr's DICT variant,
    k3_up_dict; TMG_PDICT=2 forces them even where rows barely repeat) give the same iterate as
    the dense P / Pc streams (TMG_PDICT=0), up to the kernels' different FMA contraction."""
    def make():
        if wname == "config5-L5":
            return workloads.config5(levels=5, block=27)  # config 5's block size (9 level-4 cells)
        wl = workloads.by_name("config5-L5")
        rng = np.random.default_rng(7)
        wl.tree.eps[5][...] = 10.0 ** rng.uniform(-2, 2, wl.tree.eps[5].shape)  # per-cell: few repeats
        return wl

    n = 4
    monkeypatch.setenv("TMG_PDICT", "2")
    wl1 = make()
    e1, h1 = gpu_run(wl1, n, variant)
    st = e1.weight_storage(4)
    assert st["galerkin_stored"] > 0, st  # forced (TMG_PDICT=2) even without runs
    if wname == "config5-L5":
        assert 0 < st["p_distinct"] <= st["p_rows"], st
        assert 0 < st["pc_distinct"] <= st["pc_rows"], st
    else:  # per-cell coefficients: steps / tile planes meet too many distinct rows, dense kept
        assert st["pc_distinct"] == 0 and st["p_distinct"] == 0, st
    monkeypatch.setenv("TMG_PDICT", "0")
    wl2 = make()
    e2, h2 = gpu_run(wl2, n, variant)
    assert e2.weight_storage(4)["p_distinct"] == 0 and e2.weight_storage(4)["galerkin_stored"] == 0
    np.testing.assert_allclose([s.l2h for s in h1], [s.l2h for s in h2], rtol=1e-12)
    np.testing.assert_allclose([s.linf for s in h1], [s.linf for s in h2], rtol=1e-12)
    for l in range(1, 6):
        close_u(wl1.tree.u[l], wl2.tree.u[l], 1e-12, f"level {l}")


def test_3d_weight_dictionary_default_on_blocks():
    """On blockwise-constant coefficients (config 5's structure) the default setup stores level
    ltop-1's weights (P for the restriction, the cube-owned copy for the prolongation) as
    dictionaries: far fewer distinct rows than coarse vertices / cubes; the Galerkin rows (the
    operator stream of k3_down_c) are stored in run-length form along k."""
    wl = workloads.config5(levels=5, block=27)  # config 5's block size (9 level-4 cells)
    eng, _ = gpu_run(wl, 1)
    st = eng.weight_storage(wl.tree.depth - 1)
    print(st)
    assert 0 < st["p_distinct"] <= st["p_rows"] // 4, st
    assert 0 < st["pc_distinct"] <= st["pc_rows"] // 4, st
    interior = (3 ** (wl.tree.depth - 1) - 1) ** 3
    assert 0 < st["galerkin_stored"] <= 0.6 * interior, st
