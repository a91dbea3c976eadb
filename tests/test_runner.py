"""The experiment harness (paper_1903_10367_b200.runner) against the reference's.

CPU: the configuration checks and the CSV schema of ``treemg.bench``
(tests/test_bench.py:44-57, 80-89).  GPU: whole runs through GpuEngine
reproduce the reference's CSV (tests/golden/runs/reference_runs.json, made by
tests/golden/make_runs.py from ``treemg.bench.run``, including ``pipe_*`` runs of
the reference's single-touch ``PipelineEngine``): same number of reports,
same exit status, identical integer columns, normalised residuals within
1e-12 (d-linear) / 1e-9 (BoxMG) relative.
"""

import io
import json
import os

import numpy as np
import pytest

from paper_1903_10367_b200 import runner

HERE = os.path.dirname(os.path.abspath(__file__))
RUNS = json.load(open(os.path.join(HERE, "golden", "runs", "reference_runs.json")))


def test_config_validation_messages():
    with pytest.raises(runner.ConfigError, match="setup"):
        runner.ExperimentConfig(setup="cube").validate()
    with pytest.raises(runner.ConfigError, match="k must"):
        runner.ExperimentConfig(setup="half-jump", k=9).validate()
    with pytest.raises(runner.ConfigError, match="variant"):
        runner.ExperimentConfig(variant="gauss-seidel").validate()
    with pytest.raises(runner.ConfigError, match="engine"):
        runner.ExperimentConfig(engine="gpu").validate()
    with pytest.raises(runner.ConfigError, match="pipelined"):
        runner.ExperimentConfig(engine="pipelined", variant="bpx").validate()
    runner.ExperimentConfig(engine="pipelined", variant="adafac-pi").validate()
    with pytest.raises(runner.ConfigError, match="omega"):
        runner.ExperimentConfig(omega=1.5).validate()
    with pytest.raises(runner.ConfigError, match="decile"):
        runner.ExperimentConfig(amr=True, decile=1.5).validate()
    with pytest.raises(runner.ConfigError, match="boundary_cadence"):
        runner.ExperimentConfig(amr=True, boundary_cadence=0).validate()
    runner.ExperimentConfig(amr=True).validate()
    assert runner.normalized_residuals(2.0, 3.0, (2.0, 3.0)) == (1.0, 1.0)
    assert runner.normalized_residuals(0.0, 0.0, (0.0, 0.0)) == (0.0, 0.0)


def test_csv_writer_matches_reference_format():
    ref = RUNS["schema_additive_L2"]["csv"].splitlines()
    res = runner.RunResult(2, [runner.CycleReport(0, 1.0, 1.0, 64, 0, False)])
    buf = io.StringIO()
    runner.write_csv(res, buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == ref[0] == runner.CSV_HEADER
    assert lines[1] == ref[1]


def parse(csv):
    rows = [line.split(",") for line in csv.splitlines()[1:]]
    return ([int(r[0]) for r in rows], np.array([[float(r[1]), float(r[2])] for r in rows]),
            [(int(r[3]), int(r[4]), int(r[5])) for r in rows])


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(RUNS))
def test_run_reproduces_reference_csv(name):
    case = RUNS[name]
    res = runner.run(runner.ExperimentConfig(**case["config"]))
    assert res.status == case["status"]
    buf = io.StringIO()
    runner.write_csv(res, buf)
    c1, f1, i1 = parse(buf.getvalue())
    c0, f0, i0 = parse(case["csv"])
    assert c1 == c0 and i1 == i0
    rtol = 1e-9 if case["config"].get("flavor") == "boxmg" else 1e-12
    np.testing.assert_allclose(f1, f0, rtol=rtol, atol=0)
