"""GPU parity of the spectra build and the operator apply against the
reference's own outputs (tests/golden/) — the hot-path pins of
test_toeplitz.cpp re-expressed against the B200 library, called through the
C ABI (paper_1512_06126_b200 -> libemie_cu.so)."""
import threading

import numpy as np
import pytest

import paper_1512_06126_b200 as emie
from conftest import golden

pytestmark = pytest.mark.gpu
TOEPLITZ = ["single", "tiny", "small", "large"]


def _setup(name):
    g = golden(name)
    nz = len(g["breaks"]) - 1
    sop = emie.transform_operator(g["blocks"], int(g["nx"]), int(g["ny"]), nz, float(g["omega"]))
    return g, sop


def _grid(g):
    model = emie.LayeredModel(list(g["tops"]), list(g["sigma"]))
    grid = emie.make_grid(model, list(g["breaks"]), int(g["nx"]), int(g["ny"]), float(g["hx"]),
                          float(g["hy"]))
    grid.sigma_a[...] = g["sigma_a"].reshape(grid.sigma_a.shape)
    return model, grid


@pytest.mark.parametrize("name", [f"toeplitz_{n}" for n in TOEPLITZ] + ["cfg1"])
def test_spectra_match_reference(torch_cuda, name):
    g, sop = _setup(name)
    assert (sop.ex, sop.ey, sop.qx, sop.qy) == tuple(int(x) for x in g["dims"])
    got = np.concatenate(sop.comp)
    scale = np.max(np.abs(g["spec"]))
    # test_toeplitz.cpp:214-246 gate (1e-12 of scale)
    assert np.max(np.abs(got - g["spec"])) <= 1e-12 * scale
    if name == "toeplitz_single":  # a one-point transform is the identity (:188-212)
        assert np.array_equal(got, g["blocks"].reshape(-1))


@pytest.mark.parametrize("name", [f"toeplitz_{n}" for n in TOEPLITZ] + ["cfg1"])
def test_apply_matches_reference(torch_cuda, name):
    torch = torch_cuda
    g, sop = _setup(name)
    for i, (v, want) in enumerate(zip(g["vecs"], g["applyB"])):
        got = emie.apply(sop, v)
        scale = np.max(np.abs(want))
        assert np.max(np.abs(got - want)) <= 1e-12 * scale, i
        if "denseB" in g:  # FFT apply vs the dense O(N^2) sum (:314-325)
            assert np.max(np.abs(got - g["denseB"][i])) <= 1e-12 * scale
    # batched call (nrhs fields back to back) equals the single calls bit for bit
    V = torch.from_numpy(np.ascontiguousarray(g["vecs"])).cuda()
    W = emie.apply(sop, V).cpu().numpy()
    for i, v in enumerate(g["vecs"]):
        one = emie.apply(sop, torch.from_numpy(v).cuda()).cpu().numpy()
        assert np.array_equal(W[i], one)


@pytest.mark.parametrize("name", [f"toeplitz_{n}" for n in TOEPLITZ] + ["cfg1"])
def test_system_matches_reference(torch_cuda, name):
    g, sop = _setup(name)
    model, grid = _grid(g)
    sys = emie.build_system(grid, sop)
    if "s" in g:
        s, r1, r2 = sys.diagonals()
        assert np.max(np.abs(s - g["s"])) <= 1e-14
        assert np.max(np.abs(r1 - g["r1"]) / g["r1"]) <= 1e-15
        assert np.max(np.abs(r2 - g["r2"])) <= 1e-14 * np.max(np.abs(g["r2"]))
    for v, want in zip(g["vecs"], g["applyA"]):
        got = emie.apply(sys, v)
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
        host = emie.apply_host(sys, v)
        assert np.array_equal(host, got)


def test_linearity_and_zero_map(torch_cuda):
    g, sop = _setup("toeplitz_small")  # test_toeplitz.cpp:327-347
    n = g["vecs"].shape[1]
    assert np.max(np.abs(emie.apply(sop, np.zeros(n, np.complex128)))) == 0.0
    rng = np.random.default_rng(77)
    v1 = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    v2 = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    a, b = 0.6 - 1.3j, -2.0 + 0.25j
    w1, w2 = emie.apply(sop, v1), emie.apply(sop, v2)
    wm = emie.apply(sop, a * v1 + b * v2) - (a * w1 + b * w2)
    assert np.max(np.abs(wm)) <= 1e-12 * max(np.max(np.abs(w1)), np.max(np.abs(w2)))


def test_bilinear_symmetry(torch_cuda):
    g, sop = _setup("toeplitz_small")  # test_toeplitz.cpp:366-378
    n = g["vecs"].shape[1]
    rng = np.random.default_rng(901)
    v1 = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    v2 = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    f12 = np.sum(v1 * emie.apply(sop, v2))
    f21 = np.sum(v2 * emie.apply(sop, v1))
    assert abs(f12 - f21) <= 1e-12 * abs(f12)


def test_errors(torch_cuda):
    g, sop = _setup("toeplitz_small")  # test_toeplitz.cpp:380-397
    with pytest.raises(emie.InvalidArgument):
        emie.apply(sop, np.zeros(7, np.complex128))
    with pytest.raises(emie.InvalidArgument):
        emie.transform_operator(np.zeros(0, np.complex128), 0, 0, 0)
    with pytest.raises(emie.InvalidArgument):
        emie.smooth_embedding_size(0)


def test_quadrant_budget(torch_cuda):
    g, sop = _setup("toeplitz_large")  # test_toeplitz.cpp:399-414
    assert (sop.ex, sop.ey, sop.qx, sop.qy) == (12, 9, 7, 5)
    nz = sop.nz
    assert sop.stored_complex_count() == sop.mode_count() * 2 * nz * (2 * nz + 1)


def test_concurrent_applies_bit_identical(torch_cuda):
    torch = torch_cuda
    g, sop = _setup("toeplitz_small")  # test_toeplitz.cpp:416-434
    v1 = torch.from_numpy(g["vecs"][0]).cuda()
    v2 = torch.from_numpy(g["vecs"][1]).cuda()
    w1 = emie.apply(sop, v1).cpu()
    w2 = emie.apply(sop, v2).cpu()
    res = {}

    def run(key, v):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                out = emie.apply(sop, v)
            s.synchronize()
            res[key] = out.cpu()

    t1 = threading.Thread(target=run, args=("a", v1))
    t2 = threading.Thread(target=run, args=("b", v2))
    t1.start(); t2.start(); t1.join(); t2.join()
    assert torch.equal(res["a"], w1) and torch.equal(res["b"], w2)
