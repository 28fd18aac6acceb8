"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/rhg.h declares, and its host-only entry points (parameters, band table,
argument validation) behave.  Host math is compared with the oracle."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rhg():
    import paper_1606_09481_b200 as rhg
    from paper_1606_09481_b200 import _build
    _build.build()
    return rhg


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rhg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rhg_[A-Za-z0-9_]+)\s*\(", src)))


def test_library_exports_header_symbols(rhg):
    L = rhg.lib()
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(rhg.ABI_SYMBOLS) == syms
    assert rhg.version().startswith("rhg-b200")


def test_target_radius_matches_oracle(rhg, orc):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "survey_radii.json")))
    for c in gold["configs"]:
        R = rhg.target_radius(c["n"], c["kbar"], c["gamma"])
        Ro = orc.target_radius(c["n"], c["kbar"], orc.alpha(c["gamma"]))
        assert R == pytest.approx(Ro, rel=1e-13)
        assert R == pytest.approx(c["R"], abs=2e-10)


def test_band_boundaries(rhg, orc):
    c = rhg.band_boundaries(16, 10.0, num_bands=4, band_ratio=0.9)
    assert np.allclose(c, [0, 2.9078, 5.5248, 7.8801, 10.0], atol=5e-4)
    for n, R in [(10_000, 16.7), (10_000_000, 24.9), (100_000_000, 33.9)]:
        c = rhg.band_boundaries(n, R)
        L = len(c) - 1
        # default layout (Z7): L = min(16, ceil(ln n)),
        # p = clamp(0.85 + 0.04 (ceil(ln n) - 17), 0.85, 0.95)
        lg = int(np.ceil(np.log(n)))
        assert L == min(16, lg)
        p = min(0.95, max(0.85, 0.85 + 0.04 * (lg - 17)))
        assert np.allclose(c, orc.boundaries(R, L, p), rtol=1e-12, atol=1e-12)


def test_invalid_arguments_rejected_on_host(rhg):
    L = rhg.lib()
    R = ctypes.c_double()
    assert L.rhg_target_radius(10_000, 6.0, 2.0, ctypes.byref(R)) == rhg.RHG_ERR_INVALID
    assert L.rhg_target_radius(10_000, -1.0, 3.0, ctypes.byref(R)) == rhg.RHG_ERR_INVALID
    assert L.rhg_target_radius(10_000, 6000.0, 3.0, ctypes.byref(R)) == rhg.RHG_ERR_CALIBRATION
    out = rhg.Output()
    ne = ctypes.c_uint64()
    out.num_edges = ctypes.pointer(ne)
    # n < 2, NULL outputs, bad format: rejected before any CUDA call
    assert L.rhg_generate(1, 6.0, 3.0, 1, ctypes.byref(out), None) == rhg.RHG_ERR_INVALID
    assert L.rhg_generate(1000, 6.0, 3.0, 1, ctypes.byref(out), None) == rhg.RHG_ERR_INVALID
    out.format = 7
    assert L.rhg_generate_with_radius(1000, 10.0, 1.0, 1, ctypes.byref(out), None) == \
        rhg.RHG_ERR_INVALID
    assert L.rhg_generate_with_radius(1000, 10.0, 0.5, 1, ctypes.byref(out), None) == \
        rhg.RHG_ERR_INVALID
    for s in (0, 2, 3, 4, 5, 6, 7):
        assert L.rhg_status_string(s)


def test_workspace_sizes(rhg):
    a = rhg.workspace_bytes(10_000, "csr", 60_000)
    b = rhg.workspace_bytes(1_000_000, "csr", 10_000_000)
    c = rhg.workspace_bytes(1_000_000, "csr", 10_000_000, host_buffers=True)
    assert 0 < a < b < c
    assert c - b >= 4 * 10_000_000  # host mode stages the graph on the device


def test_product_never_imports_oracle():
    """The product package must not reference oracle/ (parity rules)."""
    pkg = os.path.join(ROOT, "paper_1606_09481_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "rhg_oracle" not in txt and "liborc" not in txt, f


def test_update_workspace_and_argument_checks(rhg):
    """f1 (rhg_update_moved): the workspace grows with the row capacity and the old
    graph's size; invalid arguments are rejected on the host before any CUDA call."""
    L = rhg.lib()
    w0 = L.rhg_update_workspace_bytes(100_000, 10_000, 1_000_000, None)
    w1 = L.rhg_update_workspace_bytes(100_000, 1_000_000, 1_000_000, None)
    w2 = L.rhg_update_workspace_bytes(100_000, 1_000_000, 100_000_000, None)
    assert 0 < w0 < w1 < w2
    assert w1 - w0 >= 4 * (1_000_000 - 10_000)          # the new rows
    u = rhg.Update()
    na, nr = ctypes.c_uint64(), ctypes.c_uint64()
    u.num_added, u.num_removed = ctypes.pointer(na), ctypes.pointer(nr)
    # missing points / graph, n < 2, m > n
    assert L.rhg_update_moved(1000, None, None, 10.0, None, 0, None, None, None, None,
                              ctypes.byref(u), None) == rhg.RHG_ERR_INVALID
    assert L.rhg_update_moved(1, 8, 8, 10.0, None, 0, None, None, 8, None, ctypes.byref(u),
                              None) == rhg.RHG_ERR_INVALID
    assert L.rhg_update_moved(10, 8, 8, 10.0, 8, 11, 8, 8, 8, 8, ctypes.byref(u),
                              None) == rhg.RHG_ERR_INVALID
    assert L.rhg_update_moved(10, 8, 8, float("nan"), None, 0, None, None, 8, None,
                              ctypes.byref(u), None) == rhg.RHG_ERR_INVALID
