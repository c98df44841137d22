"""Multi-rank host logic on CPU (gloo, world_size 2): frequency sharding,
result gathering and max-over-ranks timing used by bench.py under torchrun."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

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
