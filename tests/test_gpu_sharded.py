"""Strong scaling of one grid on the GPU: the sharded
apply(SystemOperator) -- depth slabs, quadrant-mode shards of the spectra,
the two column exchanges -- run as G virtual ranks on one B200 (loopback
all-to-all) through the CUDA backend (libemie_cu.so: lateral passes, mode-range
contraction, move_planes), compared with the single-GPU apply. Every stage is
per plane / per mode / per cell, so the result is bit-identical."""
import numpy as np
import pytest

import paper_1512_06126_b200 as emie
from paper_1512_06126_b200 import configs
from paper_1512_06126_b200 import distributed as D

pytestmark = pytest.mark.gpu


def _system(cfg_id):
    cfg = configs.config(cfg_id)
    model = emie.LayeredModel(cfg.tops, cfg.sigma)
    grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
    grid.sigma_a[...] = cfg.sigma_a
    sop = emie.assemble_operator(grid, model, cfg.omega)
    return cfg, grid, sop, emie.build_system(grid, sop)


def test_mode_list_matches_plan(torch_cuda):
    cfg, grid, sop, _ = _system(1)
    plan = D.ShardPlan(cfg.nx, cfg.ny, cfg.nz, sop.ex, sop.ey, 3)
    for g in range(3):
        assert np.array_equal(emie.mode_list(sop, plan.q[g], plan.q[g + 1]), plan.modes[g])


@pytest.mark.parametrize("cfg_id,G", [(1, 1), (1, 2), (1, 3), (1, 8), (2, 4)])
def test_sharded_apply_loopback_bit_identical(torch_cuda, cfg_id, G):
    torch = torch_cuda
    cfg, grid, sop, sysop = _system(cfg_id)
    nrhs = 2
    plan = D.ShardPlan(cfg.nx, cfg.ny, cfg.nz, sop.ex, sop.ey, G)
    rng = np.random.default_rng(7 + G)
    n = 3 * cfg.cells()
    U = rng.uniform(-1, 1, (nrhs, n)) + 1j * rng.uniform(-1, 1, (nrhs, n))
    # the shards contract quadrant modes; bit identity is against the same
    # contraction order on one GPU (the octant path agrees to rounding only)
    emie.xy_symmetric(sop, disable=True)
    want = emie.apply(sysop, torch.from_numpy(U.reshape(-1)).cuda()).cpu().numpy().reshape(nrhs, n)
    shards = [D.cuda_shard(grid, sop, plan, g, nrhs) for g in range(G)]
    slabs = [torch.from_numpy(D.slab_of(U, plan, g, nrhs)).cuda() for g in range(G)]
    outs = D.loopback_apply(shards, slabs)
    got = D.join_slabs([o.cpu().numpy() for o in outs], plan, nrhs)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))
    assert np.array_equal(got, want)


def test_mode_shard_rejects_foreign_modes(torch_cuda):
    cfg, grid, sop, _ = _system(1)
    shard = emie.restrict_modes(sop, 10, 20)
    with pytest.raises(emie.InvalidArgument):
        emie.apply(shard, np.zeros(3 * cfg.cells(), np.complex128))
    with pytest.raises(emie.OutOfRange):
        emie.restrict_modes(shard, 0, 5)
