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


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("cfg_id,G", [(1, 1), (1, 2), (1, 3), (1, 8), (2, 4), (3, 2), (3, 8)])
def test_peer_exchange_loopback_bit_identical(torch_cuda, cfg_id, G, fused):
    """the transposes as peer stores (distributed.PeerExchange, csrc/peer.cu:
    IPC-shareable exchange buffers, move_planes straight into the owner's
    buffer, release/acquire flag barriers) over G virtual ranks on one GPU,
    two applies back to back (buffer and epoch reuse), with the return
    transpose fused into the contraction's epilogue and (256-point
    embeddings: config 3) the forward one into the y pass, or both as move
    kernels: bit-identical to the single-GPU apply"""
    torch = torch_cuda
    cfg, grid, sop, sysop = _system(cfg_id)
    nrhs = 2
    plan = D.ShardPlan(cfg.nx, cfg.ny, cfg.nz, sop.ex, sop.ey, G)
    emie.xy_symmetric(sop, disable=True)
    shards = [D.cuda_shard(grid, sop, plan, g, nrhs) for g in range(G)]
    xs, owns = D.peer_loopback(shards, fused=fused)
    try:
        for rep in range(2):
            rng = np.random.default_rng(70 + G + rep)
            n = 3 * cfg.cells()
            U = rng.uniform(-1, 1, (nrhs, n)) + 1j * rng.uniform(-1, 1, (nrhs, n))
            want = emie.apply(sysop, torch.from_numpy(U.reshape(-1)).cuda()).cpu().numpy().reshape(nrhs, n)
            slabs = [torch.from_numpy(D.slab_of(U, plan, g, nrhs)).cuda() for g in range(G)]
            outs = D.peer_loopback_apply(xs, slabs)
            got = D.join_slabs([o.cpu().numpy() for o in outs], plan, nrhs)
            assert np.array_equal(got, want), rep
        assert all(x.epoch == 4 for x in xs)
    finally:
        torch.cuda.synchronize()
        for o in owns:
            D.PeerExchange.free(o)


@pytest.mark.parametrize("nz,G", [(64, 2), (48, 3)])
def test_peer_exchange_deep_grid_bit_identical(torch_cuda, nz, G):
    """nz 48/64 (config 4's depth): the row-block contraction with the peer
    epilogue, G virtual ranks, bit-identical to the single-GPU apply"""
    torch = torch_cuda
    tops, sigma = [0.0, 500.0, 2500.0], [0.0, 1e-3, 10 ** -1.5, 1.0]
    breaks = list(np.linspace(600.0, 600.0 + 50.0 * nz, nz + 1))
    model = emie.LayeredModel(tops, sigma)
    nx = ny = 8
    grid = emie.make_grid(model, breaks, nx, ny, 100.0, 100.0)
    rng = np.random.default_rng(nz)
    grid.sigma_a[...] = 10.0 ** rng.uniform(-3, 0, (nz, ny, nx))
    sop = emie.assemble_operator(grid, model, 2 * np.pi * 0.5)
    emie.xy_symmetric(sop, disable=True)
    sysop = emie.build_system(grid, sop)
    nrhs = 2
    plan = D.ShardPlan(nx, ny, nz, sop.ex, sop.ey, G)
    n = 3 * nx * ny * nz
    U = rng.uniform(-1, 1, (nrhs, n)) + 1j * rng.uniform(-1, 1, (nrhs, n))
    want = emie.apply(sysop, torch.from_numpy(U.reshape(-1)).cuda()).cpu().numpy().reshape(nrhs, n)
    shards = [D.cuda_shard(grid, sop, plan, g, nrhs) for g in range(G)]
    assert shards[0].be.fused_peer_contract
    xs, owns = D.peer_loopback(shards)
    try:
        outs = D.peer_loopback_apply(xs, [torch.from_numpy(D.slab_of(U, plan, g, nrhs)).cuda() for g in range(G)])
        got = D.join_slabs([o.cpu().numpy() for o in outs], plan, nrhs)
        assert np.array_equal(got, want)
    finally:
        torch.cuda.synchronize()
        for o in owns:
            D.PeerExchange.free(o)


def test_mode_shard_rejects_foreign_modes(torch_cuda):
    cfg, grid, sop, _ = _system(1)
    shard = emie.restrict_modes(sop, 10, 20)
    with pytest.raises(emie.InvalidArgument):
        emie.apply(shard, np.zeros(3 * cfg.cells(), np.complex128))
    with pytest.raises(emie.OutOfRange):
        emie.restrict_modes(shard, 0, 5)


@pytest.mark.parametrize("G", [1, 2, 4])
def test_sharded_solve_loopback_matches_single_gpu(torch_cuda, G):
    """FGMRES on depth-sharded vectors (distributed_solve.py: the slab vector
    kernels emie_cu_vec_*, local sums summed over the ranks) against the
    single-GPU device solve on the same system: same iteration counts, same
    solution to the rounding of the rank-partitioned sums."""
    torch = torch_cuda
    from paper_1512_06126_b200 import normal_field as NF
    from paper_1512_06126_b200 import distributed_solve as DS
    cfg, grid, sop, sysop = _system(1)
    rhs = np.stack([NF.build_rhs(cfg.tops, cfg.sigma, cfg.breaks, cfg.nx, cfg.ny, cfg.omega, p).reshape(-1)
                    for p in ("x", "y")])
    nrhs = 2
    x1, reps1 = emie.fgmres_system(sysop, rhs, emie.SolverConfig(tol=1e-8, restart=40, max_iters=300))
    emie.xy_symmetric(sop, disable=True)  # the shards contract quadrant modes (same as the reference order)
    plan = D.ShardPlan(cfg.nx, cfg.ny, cfg.nz, sop.ex, sop.ey, G)
    shards = [D.cuda_shard(grid, sop, plan, g, nrhs) for g in range(G)]
    ops = [DS.CudaSlabOps() for _ in range(G)]
    slabs = [torch.from_numpy(D.slab_of(rhs, plan, g, nrhs).reshape(nrhs, -1)).cuda() for g in range(G)]

    def apply(U):
        outs = D.loopback_apply(shards, [u.reshape(-1) for u in U])
        return [o.reshape(nrhs, -1) for o in outs]

    xs, reps = DS.fgmres_sharded(apply, ops, DS.LoopbackReducer(), slabs, tol=1e-8, restart=40, max_iters=300)
    x = D.join_slabs([t.cpu().numpy() for t in xs], plan, nrhs)
    for i in range(nrhs):
        assert reps[i].status == reps1[i].status == "converged"
        assert reps[i].iterations == reps1[i].iterations
        assert np.linalg.norm(x[i] - x1[i]) <= 1e-10 * np.linalg.norm(x1[i])
        assert abs(reps[i].residual - reps1[i].residual) <= 1e-6 * reps1[i].residual


@pytest.mark.parametrize("cfg_id,G", [(1, 2), (1, 3), (0, 2)])
def test_sharded_greens_build_bit_identical(torch_cuda, cfg_id, G):
    """The Green's build split over G virtual ranks by offset (summed block
    arrays, spectra of each rank's mode shard only): the sharded apply with
    these shards equals the single-GPU apply with the full build bit for bit.
    cfg_id 0: a rectangular grid with hx != hy (no mirror)."""
    torch = torch_cuda
    if cfg_id == 0:
        model = emie.LayeredModel([0.0, 800.0, 3000.0], [0.0, 0.05, 0.01, 0.2])
        breaks = list(np.linspace(900.0, 900.0 + 40.0 * 8, 9))
        grid = emie.make_grid(model, breaks, 12, 10, 100.0, 120.0)
        grid.sigma_a[...] = 10.0 ** np.random.default_rng(3).uniform(-3, 0, grid.sigma_a.shape)
        omega = 2 * np.pi * 3.0
    else:
        cfg = configs.config(cfg_id)
        model = emie.LayeredModel(cfg.tops, cfg.sigma)
        grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
        grid.sigma_a[...] = cfg.sigma_a
        omega = cfg.omega
    sop = emie.assemble_operator(grid, model, omega)
    emie.xy_symmetric(sop, disable=True)  # shards contract quadrant modes
    sysop = emie.build_system(grid, sop)
    nrhs = 2
    plan = D.ShardPlan(grid.nx, grid.ny, grid.nz, sop.ex, sop.ey, G)
    shards_op = D.sharded_greens_build(grid, model, omega, plan, list(range(G)), D.loopback_block_sum)
    shards = [D.cuda_shard(grid, None, plan, g, nrhs, op_shard=shards_op[g]) for g in range(G)]
    rng = np.random.default_rng(9)
    n = 3 * grid.nx * grid.ny * grid.nz
    U = rng.uniform(-1, 1, (nrhs, n)) + 1j * rng.uniform(-1, 1, (nrhs, n))
    want = emie.apply(sysop, torch.from_numpy(U.reshape(-1)).cuda()).cpu().numpy().reshape(nrhs, n)
    outs = D.loopback_apply(shards, [torch.from_numpy(D.slab_of(U, plan, g, nrhs)).cuda() for g in range(G)])
    got = D.join_slabs([o.cpu().numpy() for o in outs], plan, nrhs)
    assert np.array_equal(got, want)


# ---- octant shards (ShardPlan(octant=True), Operator::shard_octant) --------
@pytest.mark.parametrize("cfg_id,G", [(1, 1), (1, 2), (1, 3), (2, 4)])
def test_octant_sharded_apply_loopback_bit_identical(torch_cuda, cfg_id, G):
    """row-aligned mode shards of an x <-> y symmetric operator contracting
    their octant rows (each block read once for a mode and its transpose):
    bit-identical to the single-GPU octant apply -- every output column is the
    same block times the same column in the same order"""
    torch = torch_cuda
    cfg, grid, sop, sysop = _system(cfg_id)
    assert emie.xy_symmetric(sop)
    nrhs = 2
    plan = D.ShardPlan(cfg.nx, cfg.ny, cfg.nz, sop.ex, sop.ey, G, octant=True)
    rng = np.random.default_rng(17 + G)
    n = 3 * cfg.cells()
    U = rng.uniform(-1, 1, (nrhs, n)) + 1j * rng.uniform(-1, 1, (nrhs, n))
    want = emie.apply(sysop, torch.from_numpy(U.reshape(-1)).cuda()).cpu().numpy().reshape(nrhs, n)
    shards = [D.cuda_shard(grid, sop, plan, g, nrhs) for g in range(G)]
    outs = D.loopback_apply(shards, [torch.from_numpy(D.slab_of(U, plan, g, nrhs)).cuda() for g in range(G)])
    got = D.join_slabs([o.cpu().numpy() for o in outs], plan, nrhs)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("cfg_id,G", [(1, 2), (1, 3), (3, 2), (3, 8)])
def test_octant_peer_exchange_loopback_bit_identical(torch_cuda, cfg_id, G, fused):
    """the peer-store exchange over octant shards (the forward y pass storing
    each mode's column into the owner of its L-shaped set; the contraction's
    peer epilogue storing the transposed modes' rows into the exchanged
    component): bit-identical to the single-GPU octant apply, twice in a row"""
    torch = torch_cuda
    cfg, grid, sop, sysop = _system(cfg_id)
    nrhs = 2
    plan = D.ShardPlan(cfg.nx, cfg.ny, cfg.nz, sop.ex, sop.ey, G, octant=True)
    shards = [D.cuda_shard(grid, sop, plan, g, nrhs) for g in range(G)]
    xs, owns = D.peer_loopback(shards, fused=fused)
    try:
        for rep in range(2):
            rng = np.random.default_rng(90 + G + rep)
            n = 3 * cfg.cells()
            U = rng.uniform(-1, 1, (nrhs, n)) + 1j * rng.uniform(-1, 1, (nrhs, n))
            want = emie.apply(sysop, torch.from_numpy(U.reshape(-1)).cuda()).cpu().numpy().reshape(nrhs, n)
            outs = D.peer_loopback_apply(xs, [torch.from_numpy(D.slab_of(U, plan, g, nrhs)).cuda() for g in range(G)])
            got = D.join_slabs([o.cpu().numpy() for o in outs], plan, nrhs)
            assert np.array_equal(got, want), rep
    finally:
        torch.cuda.synchronize()
        for o in owns:
            D.PeerExchange.free(o)


@pytest.mark.parametrize("nz,G", [(64, 2), (48, 3)])
def test_octant_peer_exchange_deep_grid_bit_identical(torch_cuda, nz, G):
    """nz 48/64: the row-block contraction, octant rows with the peer epilogue"""
    torch = torch_cuda
    tops, sigma = [0.0, 500.0, 2500.0], [0.0, 1e-3, 10 ** -1.5, 1.0]
    breaks = list(np.linspace(600.0, 600.0 + 50.0 * nz, nz + 1))
    model = emie.LayeredModel(tops, sigma)
    nx = ny = 8
    grid = emie.make_grid(model, breaks, nx, ny, 100.0, 100.0)
    rng = np.random.default_rng(nz + 1)
    grid.sigma_a[...] = 10.0 ** rng.uniform(-3, 0, (nz, ny, nx))
    sop = emie.assemble_operator(grid, model, 2 * np.pi * 0.5)
    assert emie.xy_symmetric(sop)
    sysop = emie.build_system(grid, sop)
    nrhs = 2
    plan = D.ShardPlan(nx, ny, nz, sop.ex, sop.ey, G, octant=True)
    n = 3 * nx * ny * nz
    U = rng.uniform(-1, 1, (nrhs, n)) + 1j * rng.uniform(-1, 1, (nrhs, n))
    want = emie.apply(sysop, torch.from_numpy(U.reshape(-1)).cuda()).cpu().numpy().reshape(nrhs, n)
    shards = [D.cuda_shard(grid, sop, plan, g, nrhs) for g in range(G)]
    xs, owns = D.peer_loopback(shards)
    try:
        outs = D.peer_loopback_apply(xs, [torch.from_numpy(D.slab_of(U, plan, g, nrhs)).cuda() for g in range(G)])
        got = D.join_slabs([o.cpu().numpy() for o in outs], plan, nrhs)
        assert np.array_equal(got, want)
    finally:
        torch.cuda.synchronize()
        for o in owns:
            D.PeerExchange.free(o)


@pytest.mark.parametrize("G", [2, 3])
def test_octant_sharded_greens_build_bit_identical(torch_cuda, G):
    """the offset-sharded Green's build feeding octant shards: each rank's
    shard operator checks the x <-> y symmetry on the summed blocks and
    contracts its octant rows; equal to the single-GPU build + octant apply"""
    torch = torch_cuda
    cfg = configs.config(1)
    model = emie.LayeredModel(cfg.tops, cfg.sigma)
    grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
    grid.sigma_a[...] = cfg.sigma_a
    sop = emie.assemble_operator(grid, model, cfg.omega)
    sysop = emie.build_system(grid, sop)
    nrhs = 2
    plan = D.ShardPlan(grid.nx, grid.ny, grid.nz, sop.ex, sop.ey, G, octant=True)
    shards_op = D.sharded_greens_build(grid, model, cfg.omega, plan, list(range(G)), D.loopback_block_sum)
    assert all(emie.xy_symmetric(o) for o in shards_op)
    shards = [D.cuda_shard(grid, None, plan, g, nrhs, op_shard=shards_op[g]) for g in range(G)]
    rng = np.random.default_rng(19)
    n = 3 * grid.nx * grid.ny * grid.nz
    U = rng.uniform(-1, 1, (nrhs, n)) + 1j * rng.uniform(-1, 1, (nrhs, n))
    want = emie.apply(sysop, torch.from_numpy(U.reshape(-1)).cuda()).cpu().numpy().reshape(nrhs, n)
    outs = D.loopback_apply(shards, [torch.from_numpy(D.slab_of(U, plan, g, nrhs)).cuda() for g in range(G)])
    got = D.join_slabs([o.cpu().numpy() for o in outs], plan, nrhs)
    assert np.array_equal(got, want)


def test_shard_octant_rejects_unsymmetric_or_ragged_shards(torch_cuda):
    cfg, grid, sop, _ = _system(1)
    L = emie.lib()
    ragged = emie.restrict_modes(sop, 10, 20)  # not whole rows of quadrant modes
    assert L.emie_cu_operator_shard_octant(ragged.handle, 1, None) != 0
    rows = emie.restrict_modes(sop, 0, 3 * sop.qx)
    assert L.emie_cu_operator_shard_octant(rows.handle, 1, None) == 0
    emie.xy_symmetric(sop, disable=True)
    rows2 = emie.restrict_modes(sop, 0, 3 * sop.qx)
    assert L.emie_cu_operator_shard_octant(rows2.handle, 1, None) != 0


@pytest.mark.parametrize("octant", [True, False])
def test_forward_peer_split_owner_matches_table(torch_cuda, octant):
    """the fused forward y pass with the owners computed from the plan's
    splits (emie_cu_lateral_forward_peer_split, the sharded apply's path)
    stores exactly what the per-mode owner table variant stores"""
    import ctypes
    torch = torch_cuda
    cfg, grid, sop, _ = _system(3)
    G, nrhs = 3, 2
    plan = D.ShardPlan(cfg.nx, cfg.ny, cfg.nz, sop.ex, sop.ey, G, octant=octant)
    sh = D.cuda_shard(grid, sop, plan, 1, nrhs)
    be = sh.be
    assert be.fused_peer_forward
    rng = np.random.default_rng(5)
    U = torch.from_numpy(D.slab_of(rng.uniform(-1, 1, (nrhs, 3 * cfg.cells())) + 0j, plan, 1, nrhs)).cuda()
    own = np.empty(plan.E, np.int32)
    for g, ms in enumerate(plan.modes):
        own[ms] = g
    owner = torch.from_numpy(own).cuda()
    outs = []
    for use_table in (True, False):
        dsts = [torch.zeros((nrhs, plan.E, 3 * plan.nz), dtype=torch.complex128, device="cuda") for _ in range(G)]
        dp = (ctypes.c_void_p * G)(*[d.data_ptr() for d in dsts])
        if use_table:
            rc = be.L.emie_cu_lateral_forward_peer(be.geom, ctypes.c_void_p(U.data_ptr()),
                                                   ctypes.c_void_p(be.r2.data_ptr()),
                                                   ctypes.c_void_p(owner.data_ptr()), dp, G, plan.nz,
                                                   plan.z[1], nrhs, be._st())
        else:
            be.lateral_forward_peer(U, dsts, nrhs)
            rc = 0
        assert rc == 0
        torch.cuda.synchronize()
        outs.append([d.cpu().numpy() for d in dsts])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    # each destination holds exactly its own modes' columns of this slab
    for g in range(G):
        nz0 = np.abs(outs[1][g]).sum(axis=(0, 2)) > 0
        assert set(np.nonzero(nz0)[0]) <= set(plan.modes[g].tolist())
