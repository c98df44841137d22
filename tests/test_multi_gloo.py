"""Multi-rank host logic on CPU (gloo, world_size 2): frequency sharding,
result gathering and max-over-ranks timing used by bench.py under torchrun."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from numpy_backend import NumpyBackend
from paper_1512_06126_b200.sharding import max_over_ranks, run_sweep, shard_indices


def test_shard_indices_partition():
    for world in (1, 2, 3, 8):
        for n in (1, 5, 32):
            owned = [shard_indices(n, world, r) for r in range(world)]
            flat = sorted(i for o in owned for i in o)
            assert flat == list(range(n))
    cost = [5, 1, 1, 1, 1, 1]
    owned = [shard_indices(6, 2, r, cost) for r in range(2)]
    assert sorted(owned[0] + owned[1]) == list(range(6))
    assert sum(cost[i] for i in owned[0]) == 5 and sum(cost[i] for i in owned[1]) == 5
    with pytest.raises(ValueError):
        shard_indices(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import emie_oracle as O
    freqs = list(np.logspace(-3, 2, 5))

    def job(f):
        # a tiny independent "solve" per frequency: the oracle's layer state
        m = O.LayeredModel([0.0, 400.0], [0.0, 0.01, 0.1])
        st = O.spectral_state(m, 2 * np.pi * f, [1e-3], True)
        return complex(st.p[0, 1])

    res = run_sweep(freqs, job, rank, world, dist)
    t = max_over_ranks(1.0 + rank, dist)
    if rank == 0:
        q.put((sorted(res.items()), t))
    dist.barrier()
    dist.destroy_process_group()


def test_sweep_gathers_every_frequency_gloo():
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [i for i, _ in res] == [0, 1, 2, 3, 4]
    assert t == 2.0  # max over ranks
    # serial reference
    import emie_oracle as O
    for i, v in res:
        f = np.logspace(-3, 2, 5)[i]
        m = O.LayeredModel([0.0, 400.0], [0.0, 0.01, 0.1])
        assert v == complex(O.spectral_state(m, 2 * np.pi * f, [1e-3], True).p[0, 1])


# ---- strong scaling of one grid: sharded apply -------
def _sharded_case(nx=6, ny=5, nz=4, nrhs=2, seed=11):
    import emie_oracle as O
    rng = np.random.default_rng(seed)
    nent = 2 * nz * (2 * nz + 1)
    blocks = rng.standard_normal((ny, nx, nent)) + 1j * rng.standard_normal((ny, nx, nent))
    dims, comp = O.transform_operator(blocks, nx, ny, nz)
    m = O.LayeredModel([0.0, 5000.0], [0.0, 0.01, 0.1])
    breaks = list(np.linspace(10.0, 10.0 + 50.0 * nz, nz + 1))
    sa = 10.0 ** rng.uniform(-3, 0, (nz, ny, nx))
    grid = O.make_grid(m, breaks, nx, ny, 100.0, 120.0, sa)
    diag = O.system_diagonals(grid)
    U = rng.standard_normal((nrhs, 3 * nx * ny * nz)) + 1j * rng.standard_normal((nrhs, 3 * nx * ny * nz))
    want = np.stack([O.apply_system(diag, lambda x: O.apply_spectral(comp, dims, nx, ny, nz, x), u) for u in U])
    return dims, comp, diag, U, want


def _sharded_worker(rank, world, port, q, octant=False):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1512_06126_b200 import distributed as D
    nx, ny, nz, nrhs = (6, 6, 4, 2) if octant else (6, 5, 4, 2)
    dims, comp, diag, U, _ = _sharded_case(nx, ny, nz, nrhs)
    plan = D.ShardPlan(nx, ny, nz, dims[0], dims[1], world, octant=octant)
    z0, z1 = plan.z[rank], plan.z[rank + 1]
    dslab = [np.asarray(d).reshape(nz, ny, nx)[z0:z1].reshape(-1) for d in diag]
    be = NumpyBackend(plan, rank, comp, dims, dslab)
    sysd = D.DistributedSystem(D.ShardedApply(plan, rank, be, nrhs))
    out = sysd.apply(torch.from_numpy(D.slab_of(U, plan, rank, nrhs)))
    parts = [None] * world
    dist.all_gather_object(parts, out.numpy())
    if rank == 0:
        q.put(D.join_slabs(parts, plan, nrhs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("octant", [False, True])
def test_sharded_apply_gloo_matches_full_apply(octant):
    """two processes over gloo; octant: the row-sharded octant plan (each
    rank owns the L-shaped set of quadrant modes of its octant rows)"""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q, octant)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    *_, want = _sharded_case(6, 6 if octant else 5)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))


@pytest.mark.parametrize("qy,G", [(7, 1), (7, 2), (7, 3), (129, 8), (257, 8), (5, 5)])
def test_octant_row_splits_partition_the_modes(qy, G):
    """every quadrant mode (and so every full mode) belongs to exactly one
    rank's L-shaped set; ranks hold whole rows; the sets are balanced"""
    from paper_1512_06126_b200 import distributed as D
    ex = 2 * (qy - 1)
    plan = D.ShardPlan(4, 4, 8, ex, ex, G, octant=True)
    assert plan.q == [r * plan.qx for r in plan.rows] and plan.rows[0] == 0 and plan.rows[-1] == qy
    assert all(plan.rows[g] < plan.rows[g + 1] for g in range(G))
    allq = np.sort(np.concatenate([np.asarray(qm, dtype=np.int64) for qm in plan.qmodes]))
    assert np.array_equal(allq, np.arange(plan.qx * plan.qy))
    allm = np.sort(np.concatenate(plan.modes))
    assert np.array_equal(allm, np.arange(plan.E))
    for g in range(G):  # the L-shape: larger index in the rank's rows
        for qm in plan.qmodes[g]:
            a, b = divmod(qm, plan.qx)
            assert plan.rows[g] <= max(a, b) < plan.rows[g + 1]
    if qy >= 8 * G:
        sizes = [len(qm) for qm in plan.qmodes]
        assert max(sizes) <= 1.2 * min(sizes)
    with pytest.raises(ValueError):
        D.ShardPlan(4, 4, 8, ex, ex + 2, G, octant=True)


@pytest.mark.parametrize("octant", [False, True])
@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_sharded_apply_loopback_numpy(G, octant):
    """G virtual ranks in one process (the list-transpose all-to-all)."""
    import sys
    from pathlib import Path
    import torch
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    from paper_1512_06126_b200 import distributed as D
    nx, ny, nz, nrhs = (6, 6, 4, 2) if octant else (6, 5, 4, 2)
    dims, comp, diag, U, want = _sharded_case(nx, ny, nz, nrhs)
    plan = D.ShardPlan(nx, ny, nz, dims[0], dims[1], G, octant=octant)
    # every full mode belongs to exactly one rank's list
    allm = np.sort(np.concatenate(plan.modes))
    assert np.array_equal(allm, np.arange(plan.E))
    shards = []
    for g in range(G):
        z0, z1 = plan.z[g], plan.z[g + 1]
        dslab = [np.asarray(d).reshape(nz, ny, nx)[z0:z1].reshape(-1) for d in diag]
        shards.append(D.ShardedApply(plan, g, NumpyBackend(plan, g, comp, dims, dslab), nrhs))
    outs = D.loopback_apply(shards, [torch.from_numpy(D.slab_of(U, plan, g, nrhs)) for g in range(G)])
    got = D.join_slabs([o.numpy() for o in outs], plan, nrhs)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))


@pytest.mark.parametrize("octant", [False, True])
@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_peer_exchange_loopback_numpy(G, octant):
    """The peer-store exchange plan (distributed.PeerExchange: each rank moves
    its columns straight into the owners' buffers, no pack / unpack) over G
    virtual ranks with host buffers and the NumPy stages, twice in a row
    (buffer reuse), against the oracle's full apply."""
    import sys
    from pathlib import Path
    import torch
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    from paper_1512_06126_b200 import distributed as D
    nx, ny, nz, nrhs = (6, 6, 4, 2) if octant else (6, 5, 4, 2)
    dims, comp, diag, U, want = _sharded_case(nx, ny, nz, nrhs)
    plan = D.ShardPlan(nx, ny, nz, dims[0], dims[1], G, octant=octant)
    shards = []
    for g in range(G):
        z0, z1 = plan.z[g], plan.z[g + 1]
        dslab = [np.asarray(d).reshape(nz, ny, nx)[z0:z1].reshape(-1) for d in diag]
        shards.append(D.ShardedApply(plan, g, NumpyBackend(plan, g, comp, dims, dslab), nrhs))
    xs, _ = D.peer_loopback(shards, host=True)
    for _ in range(2):
        outs = D.peer_loopback_apply(xs, [torch.from_numpy(D.slab_of(U, plan, g, nrhs)) for g in range(G)])
        got = D.join_slabs([o.numpy() for o in outs], plan, nrhs)
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
    assert all(x.epoch == 4 for x in xs)


# ---- FGMRES on depth-sharded vectors -------------------
def _solve_case(nx=6, ny=5, nz=4, nrhs=2, seed=21):
    import emie_oracle as O
    rng = np.random.default_rng(seed)
    nent = 2 * nz * (2 * nz + 1)
    blocks = 2e-3 * (rng.standard_normal((ny, nx, nent)) + 1j * rng.standard_normal((ny, nx, nent)))
    dims, comp = O.transform_operator(blocks, nx, ny, nz)
    m = O.LayeredModel([0.0, 5000.0], [0.0, 0.01, 0.1])
    breaks = list(np.linspace(10.0, 10.0 + 50.0 * nz, nz + 1))
    sa = 10.0 ** rng.uniform(-3, 0, (nz, ny, nx))
    grid = O.make_grid(m, breaks, nx, ny, 100.0, 120.0, sa)
    diag = O.system_diagonals(grid)
    B = rng.standard_normal((nrhs, 3 * nx * ny * nz)) + 1j * rng.standard_normal((nrhs, 3 * nx * ny * nz))
    A = lambda x: O.apply_system(diag, lambda v: O.apply_spectral(comp, dims, nx, ny, nz, v), x)  # noqa: E731
    want = [O.fgmres(A, b, tol=1e-10, restart=8, max_iters=200) for b in B]
    return dims, comp, diag, B, want


def _numpy_sharded_solve(G, ranks, dims, comp, diag, B, reduce, dist_apply=None, ortho="dcgs2"):
    import torch
    from paper_1512_06126_b200 import distributed as D
    from paper_1512_06126_b200 import distributed_solve as DS
    nx, ny, nz, nrhs = 6, 5, 4, B.shape[0]
    plan = D.ShardPlan(nx, ny, nz, dims[0], dims[1], G)
    shards, ops, rhs = [], [], []
    for g in ranks:
        z0, z1 = plan.z[g], plan.z[g + 1]
        dslab = [np.asarray(d).reshape(nz, ny, nx)[z0:z1].reshape(-1) for d in diag]
        shards.append(D.ShardedApply(plan, g, NumpyBackend(plan, g, comp, dims, dslab), nrhs))
        ops.append(DS.NumpySlabOps())
        rhs.append(torch.from_numpy(D.slab_of(B, plan, g, nrhs).reshape(nrhs, -1)))
    if dist_apply is None:
        def apply(U):
            outs = D.loopback_apply(shards, [u.reshape(-1) for u in U])
            return [o.reshape(nrhs, -1) for o in outs]
    else:
        sysd = D.DistributedSystem(shards[0])

        def apply(U):
            return [sysd.apply(U[0].reshape(-1)).reshape(nrhs, -1)]
    x, reps = DS.fgmres_sharded(apply, ops, reduce, rhs, tol=1e-10, restart=8, max_iters=200, ortho=ortho)
    return plan, x, reps


def _check_solve(x_full, reps, want):
    for i, (wx, wrep) in enumerate(want):
        assert reps[i].status == "converged" and wrep["status"] == "converged"
        assert abs(reps[i].iterations - wrep["iterations"]) <= 1
        assert np.linalg.norm(x_full[i] - wx) <= 1e-8 * np.linalg.norm(wx)


@pytest.mark.parametrize("G", [1, 2, 3])
@pytest.mark.parametrize("ortho", ["dcgs2", "cgs2"])
def test_sharded_solve_loopback_numpy(G, ortho):
    """both orthogonalisations (DCGS2: v_j's second projection delayed one
    step, Hessenberg column re-rotated, solution coefficients mapped back)
    against the oracle's FGMRES (MGS2, cie.cpp:117-238)"""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    from paper_1512_06126_b200 import distributed as D
    from paper_1512_06126_b200 import distributed_solve as DS
    dims, comp, diag, B, want = _solve_case()
    plan, x, reps = _numpy_sharded_solve(G, list(range(G)), dims, comp, diag, B, DS.LoopbackReducer(), ortho=ortho)
    _check_solve(D.join_slabs([t.numpy() for t in x], plan, B.shape[0]), reps, want)


def _solve_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1512_06126_b200 import distributed_solve as DS
    dims, comp, diag, B, _ = _solve_case()
    plan, x, reps = _numpy_sharded_solve(world, [rank], dims, comp, diag, B, DS.TorchReducer(), dist_apply=True)
    parts = [None] * world
    dist.all_gather_object(parts, x[0].numpy())
    if rank == 0:
        q.put((parts, [(r.status, r.iterations) for r in reps]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_solve_gloo_matches_oracle():
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    from paper_1512_06126_b200 import distributed as D
    from paper_1512_06126_b200 import SolveReport
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts, reps = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dims, comp, diag, B, want = _solve_case()
    plan = D.ShardPlan(6, 5, 4, dims[0], dims[1], 2)
    x = D.join_slabs(parts, plan, B.shape[0])
    _check_solve(x, [SolveReport(s, it) for s, it in reps], want)


def test_greens_offset_ranges_partition():
    """the sharded Green's build's split: every computed offset (all, or oi <= oj
    on square grids with hx == hy) belongs to exactly one rank's range"""
    import paper_1512_06126_b200 as emie
    from paper_1512_06126_b200 import distributed as D
    for nx, ny, hx, hy in [(16, 16, 500.0, 500.0), (12, 10, 100.0, 120.0), (8, 8, 100.0, 120.0), (1, 1, 1.0, 1.0)]:
        offs = emie.greens_offsets(nx, ny, hx, hy)
        mirror = nx == ny and hx == hy
        want = [oi * nx + oj for oi in range(ny) for oj in range(nx) if not (mirror and oi > oj)]
        assert list(offs) == want
        for G in (1, 2, 3, 8):
            rng = D.greens_offset_ranges(len(offs), G)
            assert rng[0][0] == 0 and rng[-1][1] == len(offs)
            assert all(a[1] == b[0] for a, b in zip(rng, rng[1:]))


def _greens_worker(rank, world, port, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import emie_oracle as O
    import paper_1512_06126_b200 as emie
    from paper_1512_06126_b200 import distributed as D
    nx = ny = 4
    hx = hy = 200.0
    model = O.LayeredModel([0.0, 400.0], [0.0, 0.01, 0.1])
    grid = O.make_grid(model, [0.0, 150.0, 300.0, 400.0], nx, ny, hx, hy)
    offs = emie.greens_offsets(nx, ny, hx, hy)  # oi <= oj on this square grid
    omega = 2 * np.pi / 10.0
    seen = []

    def compute(c0, c1, buf):  # the numpy oracle stands in for the device build
        for code in offs[c0:c1]:
            oi, oj = divmod(int(code), nx)
            seen.append((oi, oj))
            buf[oi, oj] = torch.from_numpy(O.block_vector(O.assemble_block(grid, omega, oi, oj)))

    (full,) = D.sharded_block_arrays(nx, ny, 3, offs, world, [rank], compute,
                                     lambda shape: torch.zeros(shape, dtype=torch.complex128),
                                     D.torch_block_sum())
    parts = [None] * world
    dist.all_gather_object(parts, (seen, full.numpy()))
    if rank == 0:
        q.put(parts)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_greens_block_sum_gloo():
    """The offset-sharded Green's build's host logic on two gloo processes:
    every computed offset is assembled by exactly one rank, and the summed
    block arrays equal the unsharded build on every rank (bitwise)."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    import emie_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_greens_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (s0, f0), (s1, f1) = parts
    assert not set(s0) & set(s1) and len(s0) + len(s1) == 10  # 4x4, oi <= oj
    assert np.array_equal(f0, f1)
    model = O.LayeredModel([0.0, 400.0], [0.0, 0.01, 0.1])
    grid = O.make_grid(model, [0.0, 150.0, 300.0, 400.0], 4, 4, 200.0, 200.0)
    for oi, oj in s0 + s1:
        want = O.block_vector(O.assemble_block(grid, 2 * np.pi / 10.0, oi, oj))
        assert np.array_equal(f0[oi, oj], want)
    untouched = [(i, j) for i in range(4) for j in range(4) if i > j]
    assert all(np.all(f0[i, j] == 0) for i, j in untouched)  # mirrors: filled on the device afterwards
