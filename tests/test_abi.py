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


def test_product_package_never_imports_the_oracle():
    """The oracle is test infrastructure: nothing under the product package may use it."""
    pkg = os.path.join(ROOT, "paper_1903_10367_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_3d_entry_points_declared_and_bound():
    decl = declared_symbols()
    for name in ("tmg3_create", "tmg3_rebuild", "tmg3_shard", "tmg3_phase", "tmg3_field",
                 "tmg3_stream", "tmg3_history", "tmg3_fused", "tmg_dim"):
        assert name in decl, name
    L = _abi.lib()
    for name in decl:
        assert getattr(L, name).argtypes is not None or name in ("tmg_last_error", "tmg_device_count"), name
