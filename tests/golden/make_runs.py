"""Golden CSVs of the reference's experiment harness (treemg.bench.run + write_csv).

Run in the build container (the reference is read-only there):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_runs.py
"""

import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from treemg.bench import ExperimentConfig, run, write_csv  # noqa: E402

CASES = {
    "schema_additive_L2": dict(setup="poisson", variant="additive", lmax=2, max_cycles=2, target=1e-30),
    "poisson_jac_L4": dict(setup="poisson", variant="adafac-jac", lmax=4, target=1e-8),
    "halfjump_pi_L3": dict(setup="half-jump", k=2, variant="adafac-pi", lmax=3, max_cycles=12,
                           target=1e-30),
    "skew_boxmg_jac_L4": dict(setup="skew", k=3, variant="adafac-jac", flavor="boxmg", lmax=4,
                              max_cycles=40, target=1e-8),
    "needle_bpx_L3": dict(setup="needle", k=1, variant="bpx", lmax=3, max_cycles=30),
    # the reference's single-touch engine (pipeline.py), SURVEY.md §8(f) item 4
    "pipe_poisson_jac_L3": dict(setup="poisson", variant="adafac-jac", lmax=3, max_cycles=15,
                                target=1e-30, engine="pipelined"),
    "pipe_halfjump_pi_L3": dict(setup="half-jump", k=2, variant="adafac-pi", lmax=3, max_cycles=10,
                                target=1e-30, engine="pipelined"),
    "pipe_skew_boxmg_additive_L3": dict(setup="skew", k=3, variant="additive", flavor="boxmg", lmax=3,
                                        max_cycles=10, target=1e-30, engine="pipelined"),
    # dynamic refinement between cycles (amr.py, bench.py:206-219), SURVEY.md §8(f) item 3
    "amr_poisson_jac_L4": dict(setup="poisson", variant="adafac-jac", lmax=4, amr=True, max_cycles=30,
                               target=1e-30),
    "amr_needle_boxmg_L5": dict(setup="needle", k=2, variant="adafac-jac", flavor="boxmg", lmax=5, amr=True,
                                max_cycles=24, target=1e-30),
    "amr_halfjump_additive_L4_c3": dict(setup="half-jump", k=1, variant="additive", lmax=4, amr=True,
                                        boundary_cadence=3, decile=0.2, max_cycles=20, target=1e-30),
}


def main():
    out = {}
    for name, kw in CASES.items():
        res = run(ExperimentConfig(**kw))
        buf = io.StringIO()
        write_csv(res, buf)
        out[name] = {"config": kw, "status": res.status, "csv": buf.getvalue()}
        print(name, res.status, len(res.reports))
    json.dump(out, open(os.path.join(HERE, "runs", "reference_runs.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
