"""The C-ABI library loads and exports every symbol include/tmg.h declares (no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1903_10367_b200 import _abi, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "tmg.h")).read()
    return sorted(set(re.findall(r"\b(tmg3?_[a-z_0-9]+)\s*\(", txt)))


def test_library_builds_and_exports_header_symbols():
    path = build.build()
    lib = ctypes.CDLL(path)
    decl = declared_symbols()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(_abi.EXPORTS)


def test_no_device_means_loud_failure_not_fallback():
    if _abi.lib().tmg_device_count() > 0:
        pytest.skip("a CUDA device is present")
    from paper_1903_10367_b200 import build_regular, GpuEngine, SolverConfig
    tree = build_regular(2)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        GpuEngine(tree, SolverConfig())


def test_config_validation_mirrors_reference():
    from paper_1903_10367_b200 import SolverConfig
    with pytest.raises(ValueError):
        SolverConfig(variant="nope")
    with pytest.raises(ValueError):
        SolverConfig(flavor="amg")
    with pytest.raises(ValueError):
        SolverConfig(omega=0.0)
    with pytest.raises(ValueError):
        SolverConfig(omega_hat=1.0)
