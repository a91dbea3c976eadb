"""Generate golden fixtures by running the REFERENCE itself (treemg, read-only).

Run in the build container only (the reference does not exist on GPU boxes):

    cd /root/repo && PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--heavy]

Each ``*.npz`` stores the inputs needed to rebuild a case without the
reference (refined sets, per-level eps, initial u, rhs) and the reference's
outputs: per-cycle ``l2h``/``linf``/``dofs``/``updates`` (solvers.py:107-115,
334-399), final ``u`` on every level, vertex kinds (spacetree.py:164-191) and,
for BoxMG cases, the P / Galerkin / R~ tables built by ``rebuild``
(solvers.py:227-250).  BASELINE-size cases regenerate their inputs from
``paper_1903_10367_b200.workloads`` (seeded) and store an input checksum.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from treemg import spacetree as rsp  # noqa: E402
from treemg.solvers import ReferenceEngine, SolverConfig  # noqa: E402

from paper_1903_10367_b200 import spacetree as psp  # noqa: E402
from paper_1903_10367_b200 import workloads  # noqa: E402

VARIANTS6 = ("additive", "additive-exp", "bpx", "afacc", "adafac-pi", "adafac-jac")
FIELDS = {"const": psp.constant_field(1.0), "jump2": psp.half_domain_jump(2),
          "skew3": psp.skew_checkerboard(3), "needle1": psp.needle_inclusion(1)}


def to_reference(tree: psp.Spacetree) -> rsp.Spacetree:
    rt = rsp.Spacetree(lmin=tree.lmin, lmax=tree.lmax)
    for l in range(tree.lmax):
        ii, jj = np.nonzero(tree.refined[l])
        if ii.size:
            rt.refine_many([rsp.CellId(l, int(i), int(j)) for i, j in zip(ii, jj)])
    for l in range(len(tree.u)):
        rt.eps[l] = tree.eps[l].copy()
        rt.u[l][...] = tree.u[l]
    rt.invalidate_kinds()
    return rt


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def save_case(name, tree, cfg_kw, rhs, cycles, store_u="all", store_tables=True,
              fas_first=True, extra_meta=None):
    t0 = time.time()
    rt = to_reference(tree)
    eng = ReferenceEngine(rt, SolverConfig(**cfg_kw))
    for l, b in rhs.items():
        eng.rhs[l] = b.copy()
    out = {}
    meta = dict(cfg=cfg_kw, cycles=cycles, lmin=tree.lmin, lmax=tree.lmax, ltop=eng.ltop,
                fas_first=fas_first, nlev_arrays=len(tree.u), store_u=store_u)
    meta.update(extra_meta or {})
    meta["inputs_sha"] = sha(np.concatenate([tree.eps[l].ravel() for l in range(len(tree.u))]
                                            + [rhs[l].ravel() for l in sorted(rhs)] + [np.zeros(0)]))
    if store_u == "all":
        for l in range(tree.lmax):
            out[f"refined_{l}"] = tree.refined[l].copy()
        for l in range(len(tree.u)):
            out[f"eps_{l}"] = tree.eps[l].copy()
            out[f"u0_{l}"] = tree.u[l].copy()
        for l, b in rhs.items():
            out[f"rhs_{l}"] = b.copy()
    if fas_first:
        eng.update_fas_state()
    hist = []
    status = "max_cycles"
    r0 = None
    for n in range(cycles):
        s = eng.advance()
        hist.append((s.l2h, s.linf, s.dofs, s.updates))
        if r0 is None:
            r0 = s.l2h
        if r0 and (s.l2h / r0 > 1e4 or s.l2h != s.l2h):
            status = "diverged"
            break
    h = np.array(hist)
    out["l2h"], out["linf"] = h[:, 0], h[:, 1]
    out["dofs"], out["updates"] = h[:, 2].astype(np.int64), h[:, 3].astype(np.int64)
    rs = eng.residual_stats()
    out["res_after"] = np.array([rs.l2h, rs.linf])
    for l in range(tree.lmin, eng.ltop + 1):
        k = rt.vertex_kinds(l)
        meta[f"kinds_sha_{l}"] = sha(k)
        meta[f"kinds_count_{l}"] = np.bincount(k.ravel(), minlength=5).tolist()
        u = rt.u[l]
        meta[f"u_sum_{l}"] = float(u.sum())
        meta[f"u_sumsq_{l}"] = float((u * u).sum())
        if store_u == "all":
            out[f"u_{l}"] = u.copy()
            out[f"kinds_{l}"] = k
        elif store_u == "sub" and l == eng.ltop:
            out[f"usub_{l}"] = u[::3, ::3].copy()
    if store_tables and cfg_kw.get("flavor") == "boxmg":
        for l, tr in eng.transfers.items():
            out[f"P_{l}"] = tr.p_table
            if tr.rtilde is not None:
                out[f"Rt_{l}"] = tr.rtilde
        for l, op in eng.ops.items():
            if hasattr(op, "tbl"):
                out[f"A_{l}"] = op.tbl
    meta["status"] = status
    meta["seconds"] = time.time() - t0
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {len(hist)} cycles, {status}, {meta['seconds']:.1f}s", flush=True)


def randomized(tree, seed):
    """Default boundary data plus a random fine iterate (tests/test_solvers.py:19-24 pattern)."""
    rng = np.random.default_rng(seed)
    L = tree.depth
    m = tree.dof_mask(L)
    tree.u[L][m] = rng.standard_normal(int(m.sum()))
    return tree


def adaptive_trees():
    a1 = psp.build_regular(2, lmax=3, field=FIELDS["jump2"])
    a1.refine_many([psp.CellId(2, i, 0) for i in range(9)] + [psp.CellId(2, 4, 4)])
    a2 = psp.build_regular(2, lmax=4, field=FIELDS["const"])
    a2.refine_many([psp.CellId(2, i, j) for i in (3, 4, 5) for j in (3, 4)] + [psp.CellId(2, 4, 0)])
    a2.refine_many([psp.CellId(3, 12, 12), psp.CellId(3, 13, 12), psp.CellId(3, 13, 13),
                    psp.CellId(3, 14, 10)])
    a3 = workloads.annulus_tree(base=2, lmax=4)
    for l in range(len(a3.eps)):
        a3.eps[l] = workloads.disc_eps(l, inside=10.0)
    return {"A1": a1, "A2": a2, "A3": a3}


def main(heavy: bool):
    # 1. regular L3: every variant x flavour x material
    for fname in ("const", "jump2", "skew3"):
        for flavor in ("geometric", "boxmg"):
            for variant in VARIANTS6:
                tree = randomized(psp.build_regular(3, field=FIELDS[fname]), 5)
                save_case(f"reg3_{fname}_{flavor}_{variant}", tree,
                          dict(variant=variant, flavor=flavor), {}, 6)
    # 2. option flags
    for fname in ("jump2", "skew3"):
        for flavor in ("geometric", "boxmg"):
            tree = randomized(psp.build_regular(3, field=FIELDS[fname]), 6)
            save_case(f"reg3_{fname}_{flavor}_jac_rtrue", tree,
                      dict(variant="adafac-jac", flavor=flavor, rtilde_true_operator=True), {}, 6)
    for flavor in ("geometric", "boxmg"):
        tree = randomized(psp.build_regular(3, field=FIELDS["skew3"]), 7)
        save_case(f"reg3_skew3_{flavor}_jac_wt03_ds05", tree,
                  dict(variant="adafac-jac", flavor=flavor, omega_tilde=0.3, damping_scale=0.5,
                       omega=0.8), {}, 6)
    tree = randomized(psp.build_regular(4, field=FIELDS["skew3"]), 8)
    save_case("reg4_skew3_boxmg_jac", tree, dict(variant="adafac-jac", flavor="boxmg"), {}, 8)
    tree = randomized(psp.build_regular(4, field=FIELDS["needle1"]), 9)
    save_case("reg4_needle1_geometric_additive", tree, dict(variant="additive"), {}, 8)
    tree = randomized(psp.build_regular(4, lmin=2, field=FIELDS["jump2"]), 10)
    save_case("reg4_lmin2_jump2_geometric_jac", tree, dict(variant="adafac-jac"), {}, 8)
    tree = randomized(psp.build_regular(2, field=FIELDS["const"]), 11)
    save_case("reg2_const_geometric_v10", tree, dict(variant="multiplicative-v10"), {}, 4)
    # 3. adaptive meshes with hanging vertices
    for tname, base in adaptive_trees().items():
        for flavor in ("geometric", "boxmg"):
            for variant in ("additive", "afacc", "adafac-pi", "adafac-jac"):
                tree = randomized(_clone(base), 12)
                save_case(f"ada{tname}_{flavor}_{variant}", tree,
                          dict(variant=variant, flavor=flavor), {}, 6)
    # 4. BASELINE configurations (seeded synthetic inputs, u0 = 0)
    wl = workloads.config2(levels=4, cycles=30)
    save_case("cfg2_L4", wl.tree, dict(variant=wl.variant, flavor=wl.flavor), wl.rhs, 30,
              fas_first=False)
    wl = workloads.config4(base=2, lmax=5, cycles=30)
    save_case("cfg4_2to5", wl.tree, dict(variant=wl.variant, flavor=wl.flavor), wl.rhs, 30,
              fas_first=False)
    wl = workloads.config1()
    save_case("cfg1_L5", wl.tree, dict(variant=wl.variant, flavor=wl.flavor), wl.rhs, wl.cycles,
              store_u="all", fas_first=False)
    wl = workloads.config2()
    save_case("cfg2_L6", wl.tree, dict(variant=wl.variant, flavor=wl.flavor), wl.rhs, wl.cycles,
              store_u="sub", store_tables=False, fas_first=False)
    if heavy:
        wl = workloads.config4()
        save_case("cfg4_4to8", wl.tree, dict(variant=wl.variant, flavor=wl.flavor), wl.rhs, 40,
                  store_u="none", store_tables=False, fas_first=False)


def _clone(tree):
    t = psp.Spacetree(lmin=tree.lmin, lmax=tree.lmax, field=tree.field)
    t.refined = [r.copy() for r in tree.refined]
    t.u = [u.copy() for u in tree.u]
    t.eps = [e.copy() for e in tree.eps]
    return t


if __name__ == "__main__":
    main("--heavy" in sys.argv)
