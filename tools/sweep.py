"""Config 5 end to end on this GPU: the frequency sweep of config 3's model
(32 frequencies log-spaced 1e-3..1e2 Hz), each an independent job -- device
Green's build, system, both plane-wave polarisations solved with FGMRES
(restart 40, tol 1e-6) -- with one JSON line per frequency and a summary.
Under torchrun, rank r takes frequencies r, r+N, ... (the bench's weak-scaling
split) and rank 0 prints the gathered summary.
    python tools/sweep.py [--max-iters 3000] [--freqs K]"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1512_06126_b200 as emie  # noqa: E402
from paper_1512_06126_b200 import configs  # noqa: E402
from paper_1512_06126_b200 import normal_field as NF  # noqa: E402
from paper_1512_06126_b200.sharding import shard_indices  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-iters", type=int, default=3000)
ap.add_argument("--freqs", type=int, default=32, help="first K frequencies of the sweep")
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
# library init as the bench does it, with the pool grown once up front: the
# builds' image batches (2 GB), the Krylov bases (2 GB at restart 40) and the
# operators otherwise make the stream-ordered pool map new memory mid-sweep
# (up to ~0.9 s for one build)
emie.warmup(reserve_bytes=8 << 30)
dist = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl")
cfg = configs.config(5)
freqs = list(cfg.freqs[:a.freqs])
model = emie.LayeredModel(cfg.tops, cfg.sigma)
grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
grid.sigma_a[...] = cfg.sigma_a
emie.warmup()
rows = []
torch.cuda.synchronize()
t_all = time.perf_counter()
for i in shard_indices(len(freqs), world, rank):
    f = freqs[i]
    omega = 2 * np.pi * f
    t0 = time.perf_counter()
    sop = emie.assemble_operator(grid, model, omega)
    sysop = emie.build_system(grid, sop)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rhs = np.stack([NF.build_rhs(cfg.tops, cfg.sigma, cfg.breaks, cfg.nx, cfg.ny, omega, p).reshape(-1)
                    for p in ("x", "y")])
    x, reps = emie.fgmres_system(sysop, torch.from_numpy(rhs.reshape(-1)).cuda(),
                                 emie.SolverConfig(tol=1e-6, restart=40, max_iters=a.max_iters))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    row = {"freq_hz": f, "greens_s": round(t1 - t0, 4), "solve_s": round(t2 - t1, 4),
           "iterations": [r.iterations for r in reps], "status": [r.status for r in reps],
           "residual": [r.residual for r in reps], "finite": bool(torch.isfinite(x).all().item())}
    rows.append(row)
    print(json.dumps(row), flush=True)
    del sop, sysop, x
torch.cuda.synchronize()
wall = time.perf_counter() - t_all
if dist:
    allrows = [None] * world
    dist.all_gather_object(allrows, rows)
    walls = [None] * world
    dist.all_gather_object(walls, wall)
    rows = [r for rs in allrows for r in rs]
    wall = max(walls)
if rank == 0:
    conv = sum(all(s == "converged" for s in r["status"]) for r in rows)
    print(json.dumps({"sweep": "config 5", "n_gpus": world, "frequencies": len(rows), "converged": conv,
                      "wall_s": round(wall, 2), "greens_s": round(sum(r["greens_s"] for r in rows), 3),
                      "solve_s": round(sum(r["solve_s"] for r in rows), 3),
                      "iterations_total": int(sum(max(r["iterations"]) for r in rows))}), flush=True)
if dist:
    dist.destroy_process_group()
