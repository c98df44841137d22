"""CPU-tier checks of the drop-in boundary: the C-ABI library builds, loads
without a GPU and exports every symbol include/emie_cu.h declares; host-side
argument validation behaves like the reference (no device compute here)."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1512_06126_b200 as emie

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "emie_cu.h").read_text()
    return sorted(set(re.findall(r"\b(emie_cu_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = emie.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_smooth_embedding_sizes():
    # test_toeplitz.cpp:171-186 (integer host logic, no device needed)
    def five_smooth(n):
        for f in (2, 3, 5):
            while n % f == 0:
                n //= f
        return n == 1
    for n in range(1, 201):
        s = emie.smooth_embedding_size(n)
        assert s >= n and five_smooth(s)
        assert not any(five_smooth(c) for c in range(n, s))
    for n, want in [(7, 8), (11, 12), (13, 15), (31, 32), (33, 36), (97, 100), (121, 125)]:
        assert emie.smooth_embedding_size(n) == want
    with pytest.raises(emie.InvalidArgument):
        emie.smooth_embedding_size(0)


def contrast_model():
    return emie.LayeredModel([0.0, 400.0], [0.0, 0.01, 0.1])


def test_grid_validation():
    # test_greens.cpp:47-72
    m = contrast_model()
    with pytest.raises(emie.InvalidArgument):
        emie.make_grid(m, [0.0, 100.0], 0, 4, 50.0, 50.0)
    with pytest.raises(emie.InvalidArgument):
        emie.make_grid(m, [0.0, 100.0], 4, 4, -1.0, 50.0)
    with pytest.raises(emie.InvalidArgument):
        emie.make_grid(m, [-50.0, 0.0], 4, 4, 50.0, 50.0)
    g = emie.make_grid(m, [0.0, 100.0, 200.0], 4, 3, 50.0, 60.0)
    assert g.nz == 2 and g.sigma_a.size == 24 and g.sigma_b[0] == 0.01
    with pytest.raises(emie.InvalidArgument):
        emie.fill_box(g, 0, 4, 0, 2, 0, 1, 1.0)
    with pytest.raises(emie.InvalidArgument):
        emie.fill_box(g, 2, 1, 0, 2, 0, 1, 1.0)
    emie.fill_box(g, 1, 2, 0, 1, 0, 0, -0.5)
    with pytest.raises(emie.InvalidArgument):
        g.validate(m)
    emie.fill_box(g, 1, 2, 0, 1, 0, 0, 0.5)
    g.validate(m)


def test_partition_and_layers():
    # test_layered.cpp:33-54
    m = emie.LayeredModel([0.0, 50.0, 150.0], [0.0, 0.02, 0.5, 0.05])
    assert [m.layer_of(z) for z in (-5.0, 0.0, 25.0, 50.0, 150.0, 1e6)] == [0, 1, 1, 2, 3, 3]
    assert m.thickness(0) == 0.0 and m.thickness(2) == 100.0 and m.thickness(3) == 0.0
    assert m.sigma_floored(0).real == 1e-9
    with pytest.raises(emie.InvalidArgument):
        emie.make_grid(m, [0.0, 60.0], 2, 2, 10.0, 10.0)
    g = emie.make_grid(m, [0.0, 25.0, 50.0, 150.0, 300.0], 2, 2, 10.0, 10.0)
    assert g.layer == [1, 1, 2, 3]


def test_contrast_coefficients():
    # SPEC.md contrast_coefficients examples; cie.cpp:9-22 errors
    a, b, gm = emie.contrast_coefficients(0.5, 0.5)
    assert b == 0 and gm == 0
    _, _, gm = emie.contrast_coefficients(10.0, 1e-3)
    assert abs(gm - 9.999 / 10.001) < 1e-15
    with pytest.raises(emie.InvalidArgument):
        emie.contrast_coefficients(1.0, 0.0)


def test_filter_params_validation():
    # test_hankel.cpp:202-210 (host-side check before any device work)
    for bad in [emie.FilterParams(0.2, 0.11), emie.FilterParams(0.2, -0.1),
                emie.FilterParams(0.2, 0.0964, 512, 200, -250), emie.FilterParams(0.2, 0.0964, 1, -1, 0)]:
        with pytest.raises(emie.InvalidArgument):
            emie.design_offset_filters(0, 0, 1.0, 1.0, bad)
