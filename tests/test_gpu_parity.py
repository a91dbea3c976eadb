"""GPU parity: libtmg.so (through GpuEngine / the C ABI) against the reference.

Every case replays a golden fixture made by running the reference itself
(tests/golden/make_golden.py) and, where useful, the CPU oracle on the same
inputs.  Tolerances (BASELINE.json north_star):

* geometric flavour: iterates bit-identical (the kernels evaluate the same
  FMA-free fp64 DAG), residual norms within 1e-13 relative (only the norm's
  summation order differs);
* BoxMG flavour: the 4x4 f-point solves cannot reproduce LAPACK's rounding
  bitwise, so per-cycle residual norms and u are checked within 1e-10
  relative;
* classification (vertex kinds) bit-exact everywhere.
"""

import numpy as np
import pytest

from golden_io import case_names, load
from oracle import mg2d
from paper_1903_10367_b200 import GpuEngine, SolverConfig, Spacetree, workloads

pytestmark = pytest.mark.gpu

GPU_CASES = [n for n in case_names(full_only=True) if not n.endswith("_v10")]
RTOL_HIST = 1e-10


def gpu_run(case, sync="eager", **kw):
    tree = case.build_tree(Spacetree)
    eng = GpuEngine(tree, SolverConfig(**case.cfg, **kw), sync=sync)
    for l, b in case.rhs().items():
        eng.rhs[l] = b
    if case.meta["fas_first"]:
        eng.update_fas_state()
    hist = eng.advance_many(len(case["l2h"]))
    eng.pull()
    return tree, eng, hist


@pytest.mark.parametrize("name", GPU_CASES)
def test_gpu_matches_reference(name):
    case = load(name)
    tree, eng, hist = gpu_run(case, sync="lazy")
    boxmg = case.cfg.get("flavor") == "boxmg"
    l2h = np.array([s.l2h for s in hist])
    linf = np.array([s.linf for s in hist])
    rt = RTOL_HIST if boxmg else 1e-13
    np.testing.assert_allclose(l2h, case["l2h"], rtol=rt, atol=0)
    np.testing.assert_allclose(linf, case["linf"], rtol=rt, atol=0)
    assert [s.dofs for s in hist] == case["dofs"].tolist()
    assert [s.updates for s in hist] == case["updates"].tolist()
    for l in case.levels_with("kinds_"):
        assert np.array_equal(eng.kinds(l), case[f"kinds_{l}"]), f"kinds level {l}"
    for l in case.levels_with("u_"):
        want = case[f"u_{l}"]
        if boxmg:
            scale = max(np.abs(want).max(), 1e-300)
            assert np.abs(tree.u[l] - want).max() <= 1e-10 * scale, f"u level {l}"
        else:
            assert np.array_equal(tree.u[l], want), f"u level {l} not bitwise equal"
    rs = eng.residual_stats()
    np.testing.assert_allclose([rs.l2h, rs.linf], case["res_after"], rtol=rt)


@pytest.mark.parametrize("name", [n for n in GPU_CASES if "boxmg" in n][:12] + ["cfg2_L4", "cfg4_2to5"])
def test_gpu_operator_tables_match_reference(name):
    """BoxMG P (operators.py:306-437), Galerkin rows (:446-478), R~ (:508-547)."""
    case = load(name)
    tree = case.build_tree(Spacetree)
    eng = GpuEngine(tree, SolverConfig(**case.cfg))
    for l in case.levels_with("P_"):
        got, want = eng.transfers[l].p_table, case[f"P_{l}"]
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-13 * max(1.0, np.abs(want).max()))
    for l in case.levels_with("A_"):
        got, want = eng.ops[l].table(), case[f"A_{l}"]
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12 * np.abs(want).max())
    for l in case.levels_with("Rt_"):
        got, want = eng.transfers[l].rtilde, case[f"Rt_{l}"]
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-13 * max(1.0, np.abs(want).max()))


def test_gpu_geometric_tables_bitwise():
    """Rediscretized stencils and diagonals are bit-identical (operators.py:190-264)."""
    case = load("reg3_skew3_geometric_adafac-jac_rtrue") if False else load("reg3_skew3_geometric_jac_rtrue")
    tree = case.build_tree(Spacetree)
    eng = GpuEngine(tree, SolverConfig(**case.cfg))
    ot = case.build_tree(mg2d.Tree)
    oe = mg2d.Engine(ot, mg2d.Config(**case.cfg))
    for l in range(eng.lmin, eng.ltop + 1):
        assert np.array_equal(eng.ops[l].table(), oe.ops[l].table())
        assert np.array_equal(eng.ops[l].diag(), oe.ops[l].diag())
        assert np.array_equal(eng.eff_eps(l), oe.eff[l])
    for l in range(eng.lmin, eng.ltop):
        assert np.array_equal(eng.transfers[l].rtilde, oe.tr[l].rt)


def test_config1_bitwise_50_cycles():
    """BASELINE config 1 (2D Poisson L5, additive, d-linear), 50 cycles: u bit-identical."""
    case = load("cfg1_L5")
    wl = workloads.config1()
    eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
    eng.rhs.update(wl.rhs)
    hist = eng.advance_many(wl.cycles)
    u = eng.fine_solution()
    assert np.array_equal(u, case[f"u_{wl.ltop}"])
    np.testing.assert_allclose([s.l2h for s in hist], case["l2h"], rtol=1e-13)


def test_config2_full_history():
    """BASELINE config 2 (L6 adaFACx BoxMG, eps blocks), 200 cycles against the reference run."""
    case = load("cfg2_L6")
    wl = workloads.config2()
    eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
    eng.rhs.update(wl.rhs)
    hist = eng.advance_many(wl.cycles)
    np.testing.assert_allclose([s.l2h for s in hist], case["l2h"], rtol=RTOL_HIST)
    np.testing.assert_allclose([s.linf for s in hist], case["linf"], rtol=RTOL_HIST)
    u = eng.fine_solution()
    want = case[f"usub_{wl.ltop}"]
    assert np.abs(u[::3, ::3] - want).max() <= 1e-10 * np.abs(want).max()
    assert abs(float(u.sum()) - case.meta[f"u_sum_{wl.ltop}"]) <= 1e-10 * np.abs(u).sum()


def test_determinism_bitwise():
    wl = workloads.config2(levels=4)
    outs = []
    for _ in range(2):
        w = workloads.config2(levels=4)
        eng = GpuEngine(w.tree, SolverConfig(variant=w.variant, flavor=w.flavor), sync="lazy")
        eng.rhs.update(w.rhs)
        h = eng.advance_many(10)
        outs.append((eng.fine_solution().copy(), [s.l2h for s in h]))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]


def test_eager_and_lazy_agree_and_single_cycles_match_batched():
    case = load("adaA2_boxmg_adafac-jac")
    t1, e1, h1 = gpu_run(case, sync="eager")
    t2 = case.build_tree(Spacetree)
    e2 = GpuEngine(t2, SolverConfig(**case.cfg), sync="eager")
    e2.update_fas_state()
    h2 = [e2.advance() for _ in range(len(case["l2h"]))]
    assert [s.l2h for s in h1] == [s.l2h for s in h2]
    for l in range(e1.lmin, e1.ltop + 1):
        assert np.array_equal(t1.u[l], t2.u[l])


def test_gpu_vs_oracle_on_box():
    """Same seeded inputs through the CPU oracle and the GPU (no fixture)."""
    wl = workloads.config4(base=2, lmax=5, cycles=12)
    ot = mg2d.Tree(lmin=wl.tree.lmin, lmax=wl.tree.lmax)
    ot.refined = [r.copy() for r in wl.tree.refined]
    ot.u = [u.copy() for u in wl.tree.u]
    ot.eps = [e.copy() for e in wl.tree.eps]
    oe = mg2d.Engine(ot, mg2d.Config(variant=wl.variant, flavor=wl.flavor))
    oe.rhs.update(wl.rhs)
    ho = [oe.advance() for _ in range(12)]
    eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
    eng.rhs.update(wl.rhs)
    hg = eng.advance_many(12)
    np.testing.assert_allclose([s.l2h for s in hg], [s.l2h for s in ho], rtol=RTOL_HIST)
    eng.pull()
    for l in range(eng.lmin, eng.ltop + 1):
        assert np.abs(wl.tree.u[l] - ot.u[l]).max() <= 1e-10 * max(np.abs(ot.u[l]).max(), 1e-300)
        assert np.array_equal(eng.kinds(l), ot.kinds(l))


def test_degenerate_collapse_raises_arithmetic_error():
    """operators.py:295-297: a degenerate lumped 2x2 system raises ArithmeticError."""
    tree = Spacetree(lmin=1, lmax=2)
    tree.refine_many([__import__("paper_1903_10367_b200").CellId(0, 0, 0)])
    tree.refine_many([__import__("paper_1903_10367_b200").CellId(1, 1, 1)])
    for l in range(len(tree.eps)):
        tree.eps[l][:] = 1.0
    tree.eps[2][:, :] = 0.0  # zero material everywhere on the fine level -> det == 0
    with pytest.raises(ArithmeticError):
        GpuEngine(tree, SolverConfig(variant="adafac-jac", flavor="boxmg"))


@pytest.mark.parametrize("name", GPU_CASES)
def test_fused_cycle_matches_reference(name):
    """SolverConfig(fused_cycle=True): the whole cycle as one persistent cooperative launch
    (k_cycle, grid barriers between the level phases; the sweep of pipeline.py:242-386 /
    solvers.py:345-395) reproduces the reference run like the level-by-level launches do --
    iterates bit-identical for the geometric flavour -- with one kernel launch per cycle."""
    case = load(name)
    tree, eng, hist = gpu_run(case, sync="lazy", fused_cycle=True)
    assert eng.launches_per_cycle() == 1
    boxmg = case.cfg.get("flavor") == "boxmg"
    rt = RTOL_HIST if boxmg else 1e-13
    np.testing.assert_allclose([s.l2h for s in hist], case["l2h"], rtol=rt, atol=0)
    np.testing.assert_allclose([s.linf for s in hist], case["linf"], rtol=rt, atol=0)
    assert [s.updates for s in hist] == case["updates"].tolist()
    for l in case.levels_with("u_"):
        want = case[f"u_{l}"]
        if boxmg:
            assert np.abs(tree.u[l] - want).max() <= 1e-10 * max(np.abs(want).max(), 1e-300), f"u level {l}"
        else:
            assert np.array_equal(tree.u[l], want), f"u level {l} not bitwise equal"


def test_fused_cycle_config4_equals_level_launches():
    """BASELINE config 4 (patch lists, hanging vertices on four levels): the one-launch cycle's
    iterate is bitwise the level-by-level launches' after 10 cycles."""
    us = []
    for fused in (False, True):
        wl = workloads.config4()
        eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor, fused_cycle=fused), sync="lazy")
        eng.rhs.update(wl.rhs)
        hist = eng.advance_many(10)
        eng.pull()
        us.append(([s.l2h for s in hist], [wl.tree.u[l].copy() for l in range(eng.lmin, eng.ltop + 1)]))
    np.testing.assert_allclose(us[0][0], us[1][0], rtol=1e-13)
    for a, b in zip(us[0][1], us[1][1]):
        assert np.array_equal(a, b)


def test_config4_full_size_against_reference():
    """BASELINE config 4 at full size (annulus 4 -> 8, eps = 100 disc, adaFACx BoxMG, 3.07 M
    fine DoFs, 34,992 hanging vertices): the same seeded inputs as the reference run
    (input SHA), bit-exact vertex classification on every level (SHA + counts) and the
    reference's residual history up to its divergence exit (bench.py:203-205)."""
    import hashlib
    import json
    case = load("cfg4_4to8")
    meta = case.meta
    wl = workloads.config4()
    tree = wl.tree
    got_sha = hashlib.sha256(np.ascontiguousarray(np.concatenate(
        [tree.eps[l].ravel() for l in range(len(tree.u))]
        + [wl.rhs[l].ravel() for l in sorted(wl.rhs)] + [np.zeros(0)])).tobytes()).hexdigest()
    assert got_sha == meta["inputs_sha"], "seeded inputs differ from the reference run"
    eng = GpuEngine(tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
    eng.rhs.update(wl.rhs)
    for l in range(eng.lmin, eng.ltop + 1):
        k = eng.kinds(l)
        assert hashlib.sha256(np.ascontiguousarray(k).tobytes()).hexdigest() == meta[f"kinds_sha_{l}"], l
        assert np.bincount(k.ravel(), minlength=5).tolist() == meta[f"kinds_count_{l}"], l
    n = len(case["l2h"])
    hist = eng.advance_many(n)
    np.testing.assert_allclose([s.l2h for s in hist], case["l2h"], rtol=1e-9)
    np.testing.assert_allclose([s.linf for s in hist], case["linf"], rtol=1e-9)
    assert [s.dofs for s in hist] == case["dofs"].tolist()
    assert [s.updates for s in hist] == case["updates"].tolist()
    # the reference stopped with EXIT_DIVERGED: normalized l2h above 1e4
    assert hist[-1].l2h / hist[0].l2h > 1e4 and meta["status"] == "diverged"
    # the refined levels ran from their patch lists: far fewer vertex tiles than the dense arrays
    # hold (level 8: the annulus covers ~7 % of the 6562^2 vertex slots), the regular levels densely
    for l in range(5, 9):
        listed, dense = eng.patch_tiles(l)
        assert 0 < listed < dense // 4, (l, listed, dense)
    assert eng.patch_tiles(4) == (0, eng.patch_tiles(4)[1])


def test_patch_lists_cover_every_existing_vertex():
    """Every vertex that exists lies in a listed tile: the run from the patch lists equals the
    reference on a small adaptive mesh for every variant (the goldens above) and, here, the
    number of listed tiles is at least the existing vertices' bounding count."""
    wl = workloads.by_name("config4-small")
    eng = GpuEngine(wl.tree, SolverConfig(variant=wl.variant, flavor=wl.flavor), sync="lazy")
    for l in range(eng.lmin, eng.ltop + 1):
        listed, dense = eng.patch_tiles(l)
        exists = int((eng.kinds(l) != 0).sum())
        th = 8 if l == eng.ltop else 2
        if listed:
            assert listed * 32 * th >= exists and listed < dense, (l, listed, dense, exists)
        else:
            assert exists == eng.kinds(l).size or (3**l + 1) ** 2 <= 1024, l
