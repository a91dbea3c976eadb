"""Dynamic refinement between cycles (paper_1903_10367_b200.amr + runner.run_loop) on the CPU.

The regrid control plane (marking, refinement, rebuild, FAS refresh) is host
logic; here it drives the CPU oracle engine (oracle/mg2d.py, bit-identical to
the reference's cycle) over the same tree object and must reproduce the
reference's own AMR runs (tests/golden/runs/reference_runs.json ``amr_*``,
made by tests/golden/make_runs.py from ``treemg.bench.run(amr=True)``): the
same report count, exit status, DoF counts, cumulative updates and regrid
cycles, normalised residuals to 1e-12 (d-linear) / 1e-9 (BoxMG: LAPACK vs LU).
The GPU engine runs the same loop in tests/test_runner.py.
"""

import io
import json
import os

import numpy as np
import pytest

from oracle import mg2d
from paper_1903_10367_b200 import amr, runner
from paper_1903_10367_b200.spacetree import CellId, build_regular

HERE = os.path.dirname(os.path.abspath(__file__))
RUNS = json.load(open(os.path.join(HERE, "golden", "runs", "reference_runs.json")))
AMR_RUNS = sorted(k for k in RUNS if k.startswith("amr_"))


class OracleOnSharedTree:
    """mg2d.Engine over an mg2d.Tree that shares its level lists with the package's Spacetree."""

    def __init__(self, tree, scfg):
        ot = mg2d.Tree(lmin=tree.lmin, lmax=tree.lmax)
        ot.refined, ot.u, ot.eps = tree.refined, tree.u, tree.eps
        self.eng = mg2d.Engine(ot, mg2d.Config(variant=scfg.variant, flavor=scfg.flavor, omega=scfg.omega,
                                               omega_tilde=scfg.omega_tilde, omega_hat=scfg.omega_hat))

    def advance(self):
        return self.eng.advance()

    def rebuild(self):
        self.eng.rebuild()

    def update_fas_state(self):
        self.eng.update_fas_state()

    def pull(self):
        pass


def parse(csv):
    rows = [line.split(",") for line in csv.splitlines()[1:]]
    return ([int(r[0]) for r in rows], np.array([[float(r[1]), float(r[2])] for r in rows]),
            [(int(r[3]), int(r[4]), int(r[5])) for r in rows])


@pytest.mark.parametrize("name", AMR_RUNS)
def test_amr_loop_on_the_oracle_reproduces_reference_csv(name):
    case = RUNS[name]
    cfg = runner.ExperimentConfig(**case["config"])
    cfg.validate()
    tree = runner.initial_tree(cfg)
    res = runner.run_loop(cfg, tree, OracleOnSharedTree(tree, cfg.solver_config()))
    assert res.status == case["status"]
    buf = io.StringIO()
    runner.write_csv(res, buf)
    c1, f1, i1 = parse(buf.getvalue())
    c0, f0, i0 = parse(case["csv"])
    assert c1 == c0 and i1 == i0
    assert any(r[2] for r in i0), "the golden run never regridded"
    rtol = 1e-9 if case["config"].get("flavor") == "boxmg" else 1e-12
    np.testing.assert_allclose(f1, f0, rtol=rtol, atol=0)


def test_policy_validation_and_empty_marks():
    with pytest.raises(ValueError):
        amr.RefinePolicy(decile=0.0)
    with pytest.raises(ValueError):
        amr.RefinePolicy(boundary_cadence=0)
    tree = build_regular(2, lmax=3)
    for u in tree.u:
        u[...] = 0.0
    # flat solution: no curvature marks; odd cycle: no boundary marks
    assert not any(m.any() for m in amr.marks_for_cycle(tree, 1).values())
    assert not any(v.any() for v in amr.curvature_vertices(tree).values())
    # even cycle: the bottom row of the finest existing level below the cap
    marks = amr.boundary_cells(tree, 0)
    assert marks[2][:, 0].all() and marks[2].sum() == 9 and not marks[1].any() and not marks[0].any()
    rep = amr.regrid(tree, marks)
    assert rep.refined_cells == 9 and rep.changed and tree.depth == 3
    assert amr.regrid(tree, amr._empty_marks(tree)).refined_cells == 0


def test_cells_around_marks_existing_unrefined_cells_only():
    tree = build_regular(1, lmax=3)
    tree.refine_many([CellId(1, 1, 1)])          # level-2 cells exist only under cell (1, 1)
    vm = {2: np.zeros((10, 10), dtype=bool)}
    vm[2][3, 3] = True                           # corner vertex of the refined patch
    cells = amr.cells_around(tree, vm)
    assert cells[2].sum() == 1 and cells[2][3, 3]
    vm[2][...] = False
    vm[2][4, 4] = True                           # interior vertex: its four cells
    assert amr.cells_around(tree, vm)[2].sum() == 4
