"""GPU parity of the 3D engine (libtmg.so through GpuEngine) against the 3D oracle.

There is no 3D reference (treemg is 2D only); the oracle ``oracle/mg3d.py``
defines the fp64 expression DAG of every 3D operation and the kernels evaluate
the same DAG, so the bar is **bitwise**: final ``u`` on every level with
``array_equal``, P and Galerkin tables with ``array_equal``; the residual
norms differ only by the reduction order of the sum of squares (rtol 1e-13).
Larger sizes are checked against committed fixtures (tests/golden3d, made by
tests/golden3d/make_golden3d.py from the oracle): per-cycle history and
SHA-256 of the final iterate.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import mg3d
from paper_1903_10367_b200 import GpuEngine, SolverConfig, workloads

pytestmark = pytest.mark.gpu

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


def check(wl, eng, hist, t, e, ohist):
    np.testing.assert_allclose([s.l2h for s in hist], [s.l2h for s in ohist], rtol=1e-13, atol=0)
    np.testing.assert_allclose([s.linf for s in hist], [s.linf for s in ohist], rtol=0, atol=0)
    assert [s.dofs for s in hist] == [s.dofs for s in ohist]
    assert [s.updates for s in hist] == [s.updates for s in ohist]
    for l in range(wl.tree.lmin, wl.tree.depth + 1):
        assert np.array_equal(wl.tree.u[l], t.u[l]), f"u level {l} not bitwise equal"


VARIANTS = ["additive", "additive-exp", "bpx", "afacc", "adafac-pi", "adafac-jac"]


@pytest.mark.parametrize("flavor", ["geometric", "boxmg"])
@pytest.mark.parametrize("variant", VARIANTS)
def test_3d_small_all_variants_bitwise(variant, flavor):
    wl = workloads.config5(levels=2, block=3) if flavor == "boxmg" else workloads.config3(levels=2)
    t, e, oh = oracle_run(wl, 6, variant, flavor)
    eng, h = gpu_run(wl, 6, variant, flavor)
    check(wl, eng, h, t, e, oh)


@pytest.mark.parametrize("name", ["config3-small", "config5-small"])
def test_3d_level3_bitwise(name):
    wl = workloads.by_name(name)
    t, e, oh = oracle_run(wl, 8)
    eng, h = gpu_run(wl, 8)
    check(wl, eng, h, t, e, oh)
    rs = eng.residual_stats()
    ors = e.residual_stats()
    np.testing.assert_allclose([rs.l2h, rs.linf], [ors.l2h, ors.linf], rtol=1e-13)


def test_3d_boxmg_tables_bitwise():
    wl = workloads.config5(levels=3)
    t, e, _ = oracle_run(wl, 0)
    eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor))
    for l in range(wl.tree.lmin, wl.tree.depth):
        assert np.array_equal(eng.transfers[l].p_table, e.tr[l].p), f"P level {l}"
        got = eng.ops[l].table().reshape(e.ops[l].tbl.shape)
        assert np.array_equal(got, e.ops[l].tbl), f"A level {l}"
    for l in range(wl.tree.lmin, wl.tree.depth + 1):
        assert np.array_equal(eng.eff_eps(l), e.eff[l]), f"eff level {l}"


def test_3d_ds0_equals_additive_and_kinds():
    wl = workloads.config5(levels=3)
    e1, h1 = gpu_run(wl, 4, "adafac-jac", damping_scale=0.0)
    wl2 = workloads.config5(levels=3)
    e2, h2 = gpu_run(wl2, 4, "additive")
    assert [s.l2h for s in h1] == [s.l2h for s in h2]
    assert np.array_equal(wl.tree.u[3], wl2.tree.u[3])
    for l in (1, 2, 3):
        assert np.array_equal(e1.kinds(l), wl.tree.vertex_kinds(l))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


FIXTURES = sorted(f[:-5] for f in os.listdir(os.path.join(HERE, "golden3d")) if f.endswith(".json"))


@pytest.mark.parametrize("name", FIXTURES)
def test_3d_fixture_history_and_sha(name):
    fx = json.load(open(os.path.join(HERE, "golden3d", name + ".json")))
    wl = workloads.by_name(fx["workload"])
    eng, h = gpu_run(wl, fx["cycles"])
    np.testing.assert_allclose([s.l2h for s in h], fx["l2h"], rtol=1e-13)
    np.testing.assert_allclose([s.linf for s in h], fx["linf"], rtol=0)
    for l, sha in fx["u_sha256"].items():
        assert _sha(wl.tree.u[int(l)]) == sha, f"u level {l}"


@pytest.mark.parametrize("ffp", ["1", "4"])
@pytest.mark.parametrize("variant", ["adafac-jac", "additive", "additive-exp", "bpx", "afacc"])
def test_3d_fused_fine_pass_equals_unfused(variant, ffp, monkeypatch):
    """The fused fine pass (pipelined schedule, BoxMG) is bit-identical to the phase-by-phase cycle."""
    n = 5
    monkeypatch.setenv("TMG_FFP", ffp)
    wl1 = workloads.by_name("config5-L4")
    e1, h1 = gpu_run(wl1, n, variant)
    monkeypatch.setenv("TMG_FFP", "0")
    wl2 = workloads.by_name("config5-L4")
    e2, h2 = gpu_run(wl2, n, variant)
    np.testing.assert_allclose([s.l2h for s in h1], [s.l2h for s in h2], rtol=1e-13)
    assert [s.linf for s in h1] == [s.linf for s in h2]
    for l in range(1, 5):
        assert np.array_equal(wl1.tree.u[l], wl2.tree.u[l]), f"level {l}"
    # state round trip: residual_stats / update_fas_state / push after a pipelined run
    np.testing.assert_allclose(e1.residual_stats().l2h, e2.residual_stats().l2h, rtol=1e-13)
    h1b = e1.advance_many(2)
    h2b = e2.advance_many(2)
    np.testing.assert_allclose([s.l2h for s in h1b], [s.l2h for s in h2b], rtol=1e-13)
    e1.pull()
    e2.pull()
    assert np.array_equal(wl1.tree.u[4], wl2.tree.u[4])


@pytest.mark.parametrize("name,variant", [("config5-small", "adafac-jac"), ("config5-L4", "adafac-jac"),
                                          ("config5-L4", "additive"), ("config5-L4", "bpx")])
def test_3d_throttled_setup_bitwise(name, variant):
    """Throttled BoxMG setup (one level per cycle, finest first) equals the oracle bitwise;
    once every level is upgraded the P and Galerkin tables equal the eager build's."""
    wl = workloads.by_name(name)
    top, lmin = wl.tree.depth, wl.tree.lmin
    n = top - lmin + 2
    t, e, oh = oracle_run(wl, n, variant, throttled=True)
    eng, h = gpu_run(wl, n, variant, throttled=True)
    check(wl, eng, h, t, e, oh)
    _, e_eager, _ = oracle_run(workloads.by_name(name), 0, variant)
    for l in range(lmin, top):
        assert np.array_equal(eng.transfers[l].p_table, e_eager.tr[l].p), f"P level {l}"
        got = eng.ops[l].table().reshape(e_eager.ops[l].tbl.shape)
        assert np.array_equal(got, e_eager.ops[l].tbl), f"A level {l}"


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


@pytest.mark.parametrize("variant,throttled", [("adafac-jac", False), ("additive", False), ("afacc", False),
                                               ("adafac-jac", True)])
def test_3d_prolongation_stream_equals_tile(variant, throttled, monkeypatch):
    """The TMA-fed finest-level prolongation (k3_up_tma over the cube-owned copy of P;
    used from depth 5 up) is bit-identical to the per-thread tiled kernel (TMG_UPQ=0),
    which the depth <= 4 tests pin to the oracle."""
    n = 4
    monkeypatch.setenv("TMG_UPQ", "1")
    wl1 = workloads.by_name("config5-L5")
    e1, h1 = gpu_run(wl1, n, variant, throttled=throttled)
    monkeypatch.setenv("TMG_UPQ", "0")
    wl2 = workloads.by_name("config5-L5")
    e2, h2 = gpu_run(wl2, n, variant, throttled=throttled)
    assert [s.l2h for s in h1] == [s.l2h for s in h2]
    assert [s.linf for s in h1] == [s.linf for s in h2]
    for l in range(1, 6):
        assert np.array_equal(wl1.tree.u[l], wl2.tree.u[l]), f"level {l}"


@pytest.mark.parametrize("variant", ["adafac-jac", "additive", "afacc"])
@pytest.mark.parametrize("wname", ["config5-L5", "random-L5"])
def test_3d_weight_dictionary_equals_dense(variant, wname, monkeypatch):
    """Level ltop-1's BoxMG weights as bitwise-verified row dictionaries (k3_smr's DICT variant,
    k3_up_dict; TMG_PDICT=2 forces them even where rows barely repeat) give the same iterate,
    bit for bit, as the dense P / Pc streams (TMG_PDICT=0)."""
    def make():
        if wname == "config5-L5":
            return workloads.config5(levels=5, block=27)  # config 5's block size (9 level-4 cells)
        wl = workloads.by_name("config5-L5")
        rng = np.random.default_rng(7)
        wl.tree.eps[5][...] = 10.0 ** rng.uniform(-2, 2, wl.tree.eps[5].shape)  # per-cell: few repeats
        return wl

    n = 4
    monkeypatch.setenv("TMG_PDICT", "2")
    monkeypatch.setenv("TMG_PDICT_SMR", "1")
    monkeypatch.setenv("TMG_PDICT_GAL", "1")
    wl1 = make()
    e1, h1 = gpu_run(wl1, n, variant)
    st = e1.weight_storage(4)
    assert 0 < st["galerkin_distinct"] <= st["galerkin_rows"], st
    if wname == "config5-L5":
        assert 0 < st["p_distinct"] <= st["p_rows"], st
        assert 0 < st["pc_distinct"] <= st["pc_rows"], st
    else:  # per-cell coefficients: steps / tile planes meet too many distinct rows, dense kept
        assert st["pc_distinct"] == 0 and st["p_distinct"] == 0, st
    monkeypatch.setenv("TMG_PDICT", "0")
    wl2 = make()
    e2, h2 = gpu_run(wl2, n, variant)
    assert e2.weight_storage(4)["p_distinct"] == 0
    assert [s.l2h for s in h1] == [s.l2h for s in h2]
    assert [s.linf for s in h1] == [s.linf for s in h2]
    for l in range(1, 6):
        assert np.array_equal(wl1.tree.u[l], wl2.tree.u[l]), f"level {l}"


@pytest.mark.parametrize("layout", [("0", "2", "0"), ("1", "2", "0"), ("1", "7", "0")])
@pytest.mark.parametrize("wname", ["config5-L5", "random-L5"])
def test_3d_smr_layouts_equal(layout, wname, monkeypatch):
    """k3_smr's thread layouts -- the default (restriction thread per coarse vertex over both
    planes and fields, 7-column smoothing groups, smoothing and restriction decoupled by named
    barriers) and the earlier ones (TMG_SMR_RV=0: two roles owning alternate planes;
    TMG_SMR_GH=2: column pairs; TMG_SMR_DEC=0: one CTA barrier per fine plane) -- give the same
    iterate bit for bit, on the dictionary (blockwise eps) and the dense (per-cell eps) weight
    paths."""
    def make():
        if wname == "config5-L5":
            return workloads.config5(levels=5, block=27)
        wl = workloads.by_name("config5-L5")
        rng = np.random.default_rng(11)
        wl.tree.eps[5][...] = 10.0 ** rng.uniform(-2, 2, wl.tree.eps[5].shape)
        return wl

    n = 4
    wl1 = make()
    e1, h1 = gpu_run(wl1, n, "adafac-jac")
    monkeypatch.setenv("TMG_SMR_RV", layout[0])
    monkeypatch.setenv("TMG_SMR_GH", layout[1])
    monkeypatch.setenv("TMG_SMR_DEC", layout[2])
    wl2 = make()
    e2, h2 = gpu_run(wl2, n, "adafac-jac")
    assert [s.l2h for s in h1] == [s.l2h for s in h2]
    assert [s.linf for s in h1] == [s.linf for s in h2]
    for l in range(1, 6):
        assert np.array_equal(wl1.tree.u[l], wl2.tree.u[l]), f"level {l}"


def test_3d_weight_dictionary_default_on_blocks():
    """On blockwise-constant coefficients (config 5's structure) the default setup stores level
    ltop-1's weights (P for the restriction, the cube-owned copy for the prolongation) as
    dictionaries: far fewer distinct rows than coarse vertices / cubes; the Galerkin rows stay
    dense unless TMG_PDICT_GAL=1."""
    wl = workloads.config5(levels=5, block=27)  # config 5's block size (9 level-4 cells)
    eng, _ = gpu_run(wl, 1)
    st = eng.weight_storage(wl.tree.depth - 1)
    print(st)
    assert 0 < st["p_distinct"] <= st["p_rows"] // 4, st
    assert 0 < st["pc_distinct"] <= st["pc_rows"] // 4, st
    assert st["galerkin_distinct"] == 0, st
