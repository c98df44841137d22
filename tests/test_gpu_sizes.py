"""GPU parity across the kernel variants the benchmark grids do not reach:
every power-of-two embedding length of the streaming FFT path (32 .. 2048),
the mixed-radix path, every nz of the FP64 tensor-core contraction (8, 16,
32), the streamed row-block contraction (nz 48 and config 4's 64) and the
DFMA contraction (other nz), single and
batched right-hand sides,
operator and system applies. The check is the numpy restatement of
apply(SpectralOperator) / apply(SystemOperator) (oracle/emie_oracle.py,
src/toeplitz.cpp:163-283, src/cie.cpp:56-73) on the same seeded operator."""
import numpy as np
import pytest

import emie_oracle as orc
import paper_1512_06126_b200 as emie

pytestmark = pytest.mark.gpu

# (nx, ny, nz): embedding lengths ex = smooth(2nx-1), ey = smooth(2ny-1)
CASES = [
    (16, 3, 8),     # ex 32 (stream), ey 5 (mixed); MMA nz 8
    (3, 32, 16),    # ex 5, ey 64; MMA nz 16
    (64, 2, 32),    # ex 128, ey 3; MMA nz 32
    (16, 16, 32),   # 32 x 32, both axes streaming
    (128, 2, 5),    # ex 256; DFMA nz 5
    (2, 128, 12),   # ey 256; DFMA nz 12
    (256, 1, 3),    # ex 512 (TMA x passes)
    (2, 256, 8),    # ey 512 (TMA y passes)
    (256, 256, 2),  # 512 x 512 (config 4's embedding), all four TMA passes
    (512, 1, 2),    # ex 1024
    (1024, 1, 1),   # ex 2048
    (10, 6, 4),     # 20 x 12, mixed radix only
    (4, 3, 64),     # streamed row blocks nz 64 (config 4's depth)
    (3, 2, 48),     # streamed row blocks nz 48
    (3, 3, 40),     # DFMA nz 40
]


def _operator(nx, ny, nz, seed):
    rng = np.random.default_rng(seed)
    nent = 2 * nz * (2 * nz + 1)
    blocks = rng.standard_normal((ny, nx, nent)) + 1j * rng.standard_normal((ny, nx, nent))
    return blocks


@pytest.mark.parametrize("nx,ny,nz", CASES)
def test_apply_sizes(torch_cuda, nx, ny, nz):
    blocks = _operator(nx, ny, nz, 1000 * nx + 10 * ny + nz)
    dims, comp = orc.transform_operator(blocks, nx, ny, nz)
    sop = emie.transform_operator(blocks, nx, ny, nz)
    assert (sop.ex, sop.ey, sop.qx, sop.qy) == tuple(dims)
    rng = np.random.default_rng(nz + 7)
    n = 3 * nx * ny * nz
    V = rng.standard_normal((3, n)) + 1j * rng.standard_normal((3, n))
    want = np.stack([orc.apply_spectral(comp, dims, nx, ny, nz, v) for v in V])
    scale = np.max(np.abs(want))
    got = np.stack([emie.apply(sop, v) for v in V])
    assert np.max(np.abs(got - want)) <= 1e-12 * scale
    # three right-hand sides in one call: contraction groups 2 + 1
    torch = torch_cuda
    W = emie.apply(sop, torch.from_numpy(np.ascontiguousarray(V)).cuda()).cpu().numpy()
    assert np.array_equal(W, got)


@pytest.mark.parametrize("nx,ny,nz", [(16, 3, 8), (64, 2, 32), (2, 128, 12), (512, 1, 2)])
def test_system_apply_sizes(torch_cuda, nx, ny, nz):
    blocks = _operator(nx, ny, nz, 77 + nx + ny + nz)
    dims, comp = orc.transform_operator(blocks, nx, ny, nz)
    sop = emie.transform_operator(blocks, nx, ny, nz)
    tops, sigma = [0.0, 5000.0], [0.0, 0.01, 0.1]
    breaks = list(np.linspace(10.0, 10.0 + 50.0 * nz, nz + 1))
    rng = np.random.default_rng(5 * nz + nx)
    sa = 10.0 ** rng.uniform(-3, 0, (nz, ny, nx))
    grid_o = orc.make_grid(orc.LayeredModel(tops, sigma), breaks, nx, ny, 100.0, 120.0, sa)
    grid = emie.make_grid(emie.LayeredModel(tops, sigma), breaks, nx, ny, 100.0, 120.0)
    grid.sigma_a[...] = sa
    sys = emie.build_system(grid, sop)
    diag = orc.system_diagonals(grid_o)
    n = 3 * nx * ny * nz
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    want = orc.apply_system(diag, lambda x: orc.apply_spectral(comp, dims, nx, ny, nz, x), v)
    got = emie.apply(sys, v)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
