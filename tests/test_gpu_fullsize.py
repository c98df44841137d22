"""Size-independent properties at the benchmark's full sizes (configs 3 and
4, BASELINE.json), on the device-built operators -- the shapes the bench
times, where an oracle comparison of every entry would take the reference
minutes per apply:

  linearity           apply(a v1 + b v2) = a apply(v1) + b apply(v2) and
                      apply(0) = 0 (test_toeplitz.cpp:327-347 at its own size)
  bilinear symmetry   v1^T A v2 = v2^T A v1 for the spectral operator
                      (reciprocity of the Green's tensor, test_toeplitz.cpp:366-378)
  nrhs batching       two fields in one call = two single calls, bit for bit
  system linearity    the same for apply(SystemOperator)

Bars as the reference's own tests: 1e-12 of the result's scale."""
import numpy as np
import pytest

import paper_1512_06126_b200 as emie
from paper_1512_06126_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[3, 4])
def built(request, torch_cuda):
    c = configs.config(request.param)
    model = emie.LayeredModel(list(c.tops), list(c.sigma))
    grid = emie.make_grid(model, list(c.breaks), c.nx, c.ny, c.hx, c.hy)
    grid.sigma_a[...] = c.sigma_a
    sop = emie.assemble_operator(grid, model, c.omega)
    sysop = emie.build_system(grid, sop)
    yield request.param, c, sop, sysop
    del sysop, sop
    torch_cuda.cuda.synchronize()


def _fields(torch, n, seed, k=2):
    g = torch.Generator(device="cuda").manual_seed(seed)
    re = torch.rand(k * n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
    im = torch.rand(k * n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
    return torch.complex(re, im)


def _maxabs(t):
    return float(t.abs().max())


def test_linearity_full_size(torch_cuda, built):
    torch = torch_cuda
    k, c, sop, sysop = built
    n = 3 * c.cells()
    v = _fields(torch, n, 100 + k)
    v1, v2 = v[:n].contiguous(), v[n:].contiguous()
    a, b = 0.6 - 1.3j, -2.0 + 0.25j
    for op in (sop, sysop):
        w1, w2 = emie.apply(op, v1), emie.apply(op, v2)
        wm = emie.apply(op, (a * v1 + b * v2).contiguous())
        scale = max(_maxabs(w1), _maxabs(w2))
        assert _maxabs(wm - (a * w1 + b * w2)) <= 1e-12 * scale * 3.0
    assert _maxabs(emie.apply(sop, torch.zeros(n, device="cuda", dtype=torch.complex128))) == 0.0


def test_bilinear_symmetry_full_size(torch_cuda, built):
    torch = torch_cuda
    k, c, sop, _ = built
    n = 3 * c.cells()
    v = _fields(torch, n, 200 + k)
    v1, v2 = v[:n].contiguous(), v[n:].contiguous()
    f12 = complex(torch.sum(v1 * emie.apply(sop, v2)))
    f21 = complex(torch.sum(v2 * emie.apply(sop, v1)))
    # the sums run over 1.6e6 (config 3) / 1.3e7 (config 4) terms: rounding
    # of the sums themselves, relative to the sum of the terms' moduli
    w2 = emie.apply(sop, v2)
    mag = float(torch.sum((v1 * w2).abs()))
    assert abs(f12 - f21) <= 1e-12 * mag


def test_nrhs_batch_bit_identical_full_size(torch_cuda, built):
    torch = torch_cuda
    k, c, _, sysop = built
    n = 3 * c.cells()
    v = _fields(torch, n, 300 + k)
    both = emie.apply(sysop, v)
    one = emie.apply(sysop, v[:n].contiguous())
    two = emie.apply(sysop, v[n:].contiguous())
    assert torch.equal(both[:n], one) and torch.equal(both[n:], two)
