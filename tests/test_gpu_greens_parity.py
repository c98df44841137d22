"""Green's-block parity at the benchmark configurations (device vs the
reference's assemble_block, src/greens.cpp:150-221), with the bar tied to the
reference's own arithmetic.

The reference's blocks are determined only to the precision its own double
evaluation allows (oracle/ref_envelope.py): the filter sums are
ill-conditioned (V1 + V3 cancels up to 13 digits as lambda -> 0, V2 + V5 as
lambda -> inf; tests/test_gpu_vfunctions.py measures both), so the reference
moves by 1e-6 (config 1) to 7e-5 (config 3) of the block maximum when the same
sources are compiled with FMA contraction. Per block, the envelope is the
largest move of the reference under {hx + 1 ulp, hy + 1 ulp, FMA build}; the
device block must lie within ENV_FACTOR times it. The small-lambda noise of
V1 + V3 is a lambda-independent constant per interval (eta is exactly
sqrt(-i omega mu0 sigma) once lambda^2 is below its ulp), so every block of a
configuration draws on the same few rounding constants: the per-configuration
median ratio is one random draw, hence the factor. The well-conditioned
components (xz, yz: no cancelling sums) are held to 1e-10 of the block max.

Offsets: every computed offset of config 1; deterministic samples (diagonal,
edges, near and far) of configs 2-4, evaluated on the device by
emie.assemble_block (the signed-offset entry, the kernels of the full build)
and, for configs 1-3, also read from the full device build (mirror and
diagonal symmetrisation included)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1512_06126_b200 as emie
import ref_envelope as RE
from paper_1512_06126_b200 import configs

pytestmark = pytest.mark.gpu
ENV_FACTOR = 4.0
MEDIAN_FACTOR = 3.5


def _offsets(k, nx, ny):
    if k == 1:
        return [(i, j) for i in range(ny) for j in range(nx) if i <= j] + [(-3, 5), (4, -7), (-15, -15)]
    rng = np.random.default_rng(100 + k)
    pts = {(0, 0), (0, 1), (1, 1), (0, nx - 1), (ny - 1, nx - 1), (ny - 1, 0), (2, 3), (3, 2), (-2, 5), (5, -9)}
    n = {2: 48, 3: 32, 4: 14}[k]
    while len(pts) < n:
        i, j = rng.integers(0, nx, 2)
        pts.add((int(min(i, j)), int(max(i, j))))
    return sorted(pts)


def _comp_slices(nz):
    nt, nf = nz * (nz + 1) // 2, nz * nz
    return {"xz": slice(4 * nt, 4 * nt + nf), "yz": slice(4 * nt + nf, 4 * nt + 2 * nf)}


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_blocks_within_reference_envelope(torch_cuda, k):
    c = configs.config(k)
    model = emie.LayeredModel(list(c.tops), list(c.sigma))
    grid = emie.make_grid(model, list(c.breaks), c.nx, c.ny, c.hx, c.hy)
    offs = np.array(_offsets(k, c.nx, c.ny))
    dev = emie.assemble_block(grid, model, c.omega, offs[:, 0], offs[:, 1])
    ref = RE.reference_blocks(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega, offs)
    scale = np.max(np.abs(ref["ref"]), axis=1)
    env = RE.envelope(ref)
    err = np.max(np.abs(dev - ref["ref"]), axis=1) / scale
    ratio = err / env
    worst = int(np.argmax(ratio))
    msg = (f"cfg{k}: device error max {err.max():.2e} median {np.median(err):.2e}; envelope median "
           f"{np.median(env):.2e}; ratio max {ratio.max():.2f} (offset {tuple(offs[worst])}) median "
           f"{np.median(ratio):.2f}")
    print(msg)
    assert np.all(ratio <= ENV_FACTOR), msg
    assert np.median(ratio) <= MEDIAN_FACTOR, msg
    for name, sl in _comp_slices(c.nz).items():  # no cancelling sums: tight
        e = np.max(np.abs(dev[:, sl] - ref["ref"][:, sl]), axis=1) / scale
        assert e.max() <= 1e-10, f"cfg{k} {name}: {e.max():.2e}"
    if k < 4:  # the full build's stored blocks (oi <= oj computed; the rest mirrored)
        op = emie.assemble_operator(grid, model, c.omega, keep_blocks=True)
        allb = op.blocks().reshape(c.ny, c.nx, -1)
        sel = [(i, (a, b)) for i, (a, b) in enumerate(offs) if 0 <= a < b]
        full = np.stack([allb[a, b] for _, (a, b) in sel])
        idx = [i for i, _ in sel]
        # the full build runs the fused kernel or (large builds) the split
        # chunk-image kernels with images shared by offsets at equal R: the
        # same formulas in another kernel, so rounding-level agreement with
        # assemble_block, and the same bar against the reference
        d = np.max(np.abs(full - dev[idx]), axis=1) / scale[idx]
        assert d.max() <= 1e-7, f"full build vs assemble_block: {d.max():.2e}"
        rf = np.max(np.abs(full - ref["ref"][idx]), axis=1) / scale[idx] / env[idx]
        assert np.all(rf <= ENV_FACTOR), f"cfg{k} full build: envelope ratio {rf.max():.2f}"
