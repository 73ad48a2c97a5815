"""CPU-side checks of the C ABI: the library loads, exports every symbol
include/rcb.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1403_0240_b200", "librcseg_b200.so")


def header_symbols():
    text = open(os.path.join(ROOT, "include", "rcb.h")).read()
    return sorted(set(re.findall(r"\b(rcb_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = header_symbols()
    for must in ("rcb_sobolev_filter", "rcb_scan_contour", "rcb_delta_external_batch",
                 "rcb_delta_internal_batch", "rcb_evaluate_total", "rcb_engine_create",
                 "rcb_engine_iterate"):
        assert must in syms


def test_library_exports_every_header_symbol():
    if not os.path.exists(LIB):
        pytest.fail("librcseg_b200.so not built (run make)")
    lib = ctypes.CDLL(LIB)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.rcb_version() >= 100


def test_binding_covers_header():
    from paper_1403_0240_b200 import _lib
    assert set(header_symbols()) == set(_lib.SIGNATURES)


def test_no_gpu_means_loud_failure():
    from paper_1403_0240_b200 import _lib
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    import paper_1403_0240_b200 as P
    with pytest.raises(RuntimeError):
        P.sobolev_filter(np.array([[1, 1]]), [1], [0], [1.0], P.SobolevParams())
    with pytest.raises(RuntimeError):
        P.RegionCompetition(np.zeros((4, 4)), np.zeros((4, 4), np.int32), P.EnergyConfig())


def test_validation_matches_reference_errors():
    import paper_1403_0240_b200 as P
    with pytest.raises(ValueError):
        P.EnergyConfig(region_model="blob")
    with pytest.raises(ValueError):
        P.SobolevParams(length_scale=0.0)
    with pytest.raises(ValueError):
        P.OptimizerConfig(move_budget=1.5)
    with pytest.raises(ValueError):
        P.Connectivity(2, 6)
    with pytest.raises(ValueError):
        P.kernel_eval(6.1, P.SobolevParams())
    p = P.SobolevParams()
    assert abs(P.kernel_eval(0.0, p) - 0.25) < 1e-12
    assert abs(P.kernel_eval(3.0, p) - 0.0625) < 1e-12


def test_weight_table_matches_reference_golden():
    from paper_1403_0240_b200.sobolev import weight_table
    from tests.conftest import golden
    g = golden("kernel.npz")
    k = 0
    while f"E{k}" in g:
        E, eps = g[f"E{k}"]
        assert np.array_equal(weight_table(float(E), float(eps)), g[f"w{k}"])
        k += 1


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1403_0240_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in src and "import oracle" not in src, f
                assert "rc_oracle" not in src, f
