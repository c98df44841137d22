"""GPU parity of the octant contraction: on a square grid whose compressed
blocks are exactly x <-> y symmetric (block(oj, oi) = block(oi, oj) with
xx <-> yy and xz <-> yz), the contraction reads only the modes qmx <= qmy
and serves each transposed mode from the same block with the x and y thirds
exchanged (operator.cu, contract_mma_kernel<NZ, true>; for other depths the
DFMA contract_kernel runs the two halves of an octant item on neighbouring
warp groups). The check is the
oracle's apply over every quadrant mode (oracle/emie_oracle.py, which follows
src/toeplitz.cpp:163-283 and src/cie.cpp:56-73 and uses no symmetry), plus the
same operator with the octant path switched off."""
import numpy as np
import pytest

import emie_oracle as orc
import paper_1512_06126_b200 as emie

pytestmark = pytest.mark.gpu


def _swap_xy(b, nz):
    """entries of one compressed block with xx <-> yy and xz <-> yz exchanged"""
    ntri, nfull = nz * (nz + 1) // 2, nz * nz
    o = b.copy()
    o[..., :ntri], o[..., ntri:2 * ntri] = b[..., ntri:2 * ntri], b[..., :ntri]
    x0, y0 = 4 * ntri, 4 * ntri + nfull
    o[..., x0:y0], o[..., y0:] = b[..., y0:], b[..., x0:y0]
    return o


def _symmetric_blocks(n, nz, seed):
    rng = np.random.default_rng(seed)
    nent = 2 * nz * (2 * nz + 1)
    b = rng.standard_normal((n, n, nent)) + 1j * rng.standard_normal((n, n, nent))
    for oi in range(n):
        for oj in range(oi + 1, n):
            b[oj, oi] = _swap_xy(b[oi, oj], nz)
        ntri, nfull = nz * (nz + 1) // 2, nz * nz
        b[oi, oi, ntri:2 * ntri] = b[oi, oi, :ntri]
        b[oi, oi, 4 * ntri + nfull:] = b[oi, oi, 4 * ntri:4 * ntri + nfull]
    return b


@pytest.mark.parametrize("n,nz", [(16, 8), (12, 16), (8, 32), (20, 32), (3, 8), (1, 16),
                                  (6, 5), (9, 12), (4, 48), (5, 64)])  # DFMA (nz 5, 12), streamed rows (48, 64)
def test_octant_apply_matches_oracle(torch_cuda, n, nz):
    blocks = _symmetric_blocks(n, nz, 31 * n + nz)
    dims, comp = orc.transform_operator(blocks, n, n, nz)
    sop = emie.transform_operator(blocks, n, n, nz)
    assert emie.xy_symmetric(sop)
    rng = np.random.default_rng(n + nz)
    V = rng.standard_normal((3, 3 * n * n * nz)) + 1j * rng.standard_normal((3, 3 * n * n * nz))
    want = np.stack([orc.apply_spectral(comp, dims, n, n, nz, v) for v in V])
    scale = np.max(np.abs(want))
    got = np.stack([emie.apply(sop, v) for v in V])
    assert np.max(np.abs(got - want)) <= 1e-12 * scale
    # batched right-hand sides (contraction groups 2 + 1) give the same columns
    torch = torch_cuda
    W = emie.apply(sop, torch.from_numpy(np.ascontiguousarray(V)).cuda()).cpu().numpy()
    assert np.array_equal(W, got)
    # the quadrant contraction on the same spectra agrees to rounding
    assert not emie.xy_symmetric(sop, disable=True)
    full = np.stack([emie.apply(sop, v) for v in V])
    assert np.max(np.abs(full - got)) <= 1e-13 * scale


def test_octant_requires_exact_symmetry(torch_cuda):
    n, nz = 8, 16
    b = _symmetric_blocks(n, nz, 5)
    b[3, 5, 7] += 1e-15 * abs(b[3, 5, 7])  # one entry off by an ulp-sized amount
    assert not emie.xy_symmetric(emie.transform_operator(b, n, n, nz))
    b = _symmetric_blocks(n, nz, 6)
    b[2, 2, 0] = b[2, 2, 0] * (1 + 1e-15)  # diagonal offset: xx != yy
    assert not emie.xy_symmetric(emie.transform_operator(b, n, n, nz))
    # rectangular grids never take the octant path
    rng = np.random.default_rng(7)
    nent = 2 * nz * (2 * nz + 1)
    r = rng.standard_normal((4, 6, nent)) + 0j
    assert not emie.xy_symmetric(emie.transform_operator(r, 6, 4, nz))


def _greens_grid(n, nz, hx, hy):
    model = emie.LayeredModel([0.0, 800.0, 3000.0], [0.0, 0.05, 0.01, 0.2])
    breaks = list(np.linspace(900.0, 900.0 + 40.0 * nz, nz + 1))
    return model, emie.make_grid(model, breaks, n, n, hx, hy)


def test_greens_build_square_grid_is_exactly_symmetric(torch_cuda):
    """the device Green's build on a square grid with hx == hy mirrors the
    offsets oi > oj (greens.cu, mirror_blocks_kernel); its diagonal offsets
    must then also be exactly symmetric for the octant contraction to apply"""
    model, grid = _greens_grid(12, 8, 100.0, 100.0)
    sop = emie.assemble_operator(grid, model, 2 * np.pi * 3.0, keep_blocks=True)
    assert emie.xy_symmetric(sop)
    blocks = sop.blocks()
    dims, comp = orc.transform_operator(blocks, 12, 12, 8)
    rng = np.random.default_rng(3)
    v = rng.standard_normal(3 * 12 * 12 * 8) + 1j * rng.standard_normal(3 * 12 * 12 * 8)
    want = orc.apply_spectral(comp, dims, 12, 12, 8, v)
    got = emie.apply(sop, v)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
    # hx != hy: no mirror, no octant
    model, grid = _greens_grid(12, 8, 100.0, 120.0)
    assert not emie.xy_symmetric(emie.assemble_operator(grid, model, 2 * np.pi * 3.0))


def test_octant_system_apply(torch_cuda):
    n, nz = 10, 16
    blocks = _symmetric_blocks(n, nz, 11)
    dims, comp = orc.transform_operator(blocks, n, n, nz)
    sop = emie.transform_operator(blocks, n, n, nz)
    assert emie.xy_symmetric(sop)
    tops, sigma = [0.0, 5000.0], [0.0, 0.01, 0.1]
    breaks = list(np.linspace(10.0, 10.0 + 50.0 * nz, nz + 1))
    rng = np.random.default_rng(12)
    sa = 10.0 ** rng.uniform(-3, 0, (nz, n, n))
    grid_o = orc.make_grid(orc.LayeredModel(tops, sigma), breaks, n, n, 100.0, 100.0, sa)
    grid = emie.make_grid(emie.LayeredModel(tops, sigma), breaks, n, n, 100.0, 100.0)
    grid.sigma_a[...] = sa
    sys = emie.build_system(grid, sop)
    diag = orc.system_diagonals(grid_o)
    v = rng.standard_normal(3 * n * n * nz) + 1j * rng.standard_normal(3 * n * n * nz)
    want = orc.apply_system(diag, lambda x: orc.apply_spectral(comp, dims, n, n, nz, x), v)
    got = emie.apply(sys, v)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))


@pytest.mark.parametrize("nz,nrhs", [(8, 2), (16, 1), (5, 3), (8, 7)])
def test_host_apply_matches_device_apply(torch_cuda, nz, nrhs):
    """host buffers through emie_cu_apply_system_host on a 256-point
    embedding (the bench's e2e path: per-rhs pipeline over separate upload /
    download streams, nrhs = 1 contractions with packed octant columns; 7
    fields cycle the three-slot device ring twice) equal the device-resident
    batched apply bit for bit"""
    torch = torch_cuda
    n = 128
    blocks = _symmetric_blocks(n, nz, 40 + nz)
    sop = emie.transform_operator(blocks, n, n, nz)
    tops, sigma = [0.0, 5000.0], [0.0, 0.01, 0.1]
    breaks = list(np.linspace(10.0, 10.0 + 50.0 * nz, nz + 1))
    rng = np.random.default_rng(nz)
    grid = emie.make_grid(emie.LayeredModel(tops, sigma), breaks, n, n, 100.0, 100.0)
    grid.sigma_a[...] = 10.0 ** rng.uniform(-3, 0, (nz, n, n))
    sys = emie.build_system(grid, sop)
    N = 3 * n * n * nz
    V = rng.standard_normal((nrhs, N)) + 1j * rng.standard_normal((nrhs, N))
    dev = emie.apply(sys, torch.from_numpy(V.reshape(-1)).cuda()).cpu().numpy().reshape(nrhs, N)
    host = emie.apply_host(sys, V).reshape(nrhs, N)
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("n,nz", [(64, 16), (64, 32), (16, 64)])
def test_repeated_contractions_bit_identical(torch_cuda, n, nz):
    """the pipelined contractions refill SMEM stages with TMA right after the
    consumers release them; repeated launches on the same spectrum must agree
    bit for bit (a missing generic->async proxy fence before the release once
    let a refill overtake the last reads: ~10 % of nz = 16 launches differed)"""
    import ctypes
    torch = torch_cuda
    blocks = _symmetric_blocks(n, nz, 5)
    sop = emie.transform_operator(blocks, n, n, nz)
    L = emie.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    nrhs, E = 2, sop.ex * sop.ey
    g = torch.Generator(device="cuda").manual_seed(3)
    S0 = torch.complex(torch.rand(nrhs * E * 3 * nz, device="cuda", dtype=torch.float64, generator=g),
                       torch.rand(nrhs * E * 3 * nz, device="cuda", dtype=torch.float64, generator=g))
    ref = None
    for _ in range(20):
        S = S0.clone()
        emie._check(L.emie_cu_contract_modes(sop.handle, ctypes.c_void_p(S.data_ptr()), nrhs, 0, sop.qx * sop.qy, st))
        if ref is None:
            ref = S
        else:
            assert torch.equal(ref, S)
