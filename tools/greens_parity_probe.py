"""Green's-block parity diagnostics (GPU box): device build vs the reference.

For sampled offsets of configs 1-4 this records, per block,
  dev    the device block (full device build, keep_blocks)
  ref    the reference's assemble_block (oracle/_ref)
  refx   the reference with hx moved by one ulp (its own conditioning)
  refy   the same for hy
  refw   the reference's accumulation with the DEVICE filter weights
so that |dev - ref| splits into the filter design (|refw - ref|) and the
lambda accumulation (|dev - refw|), each against the reference's own 1-ulp
sensitivity. Output: gpurun_out/greens_probe_cfgN.npz + a printed summary.

    python tools/greens_parity_probe.py 1 2 3
"""
from __future__ import annotations

import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import paper_1512_06126_b200 as emie  # noqa: E402
import ref_binding as R  # noqa: E402
from paper_1512_06126_b200 import configs  # noqa: E402


def sample_offsets(nx, ny, k):
    if k == 1:
        return [(i, j) for i in range(ny) for j in range(nx) if i <= j]
    rng = np.random.default_rng(7 + k)
    pts = {(0, 0), (0, 1), (1, 1), (0, nx - 1), (ny - 1, nx - 1), (1, nx - 1), (0, nx // 2), (2, 3), (5, 5)}
    n = {2: 60, 3: 40, 4: 16}[k]
    while len(pts) < n:
        i, j = sorted(rng.integers(0, nx, 2))
        pts.add((int(i), int(j)))
    return sorted(pts)


def block_err(a, b, scale):
    return float(np.max(np.abs(a - b)) / scale)


def run(k):
    c = configs.config(k)
    model = emie.LayeredModel(list(c.tops), list(c.sigma))
    grid = emie.make_grid(model, list(c.breaks), c.nx, c.ny, c.hx, c.hy)
    offs = sample_offsets(c.nx, c.ny, k)
    t0 = time.time()
    if k < 4:
        op = emie.assemble_operator(grid, model, c.omega, keep_blocks=True)
        allb = op.blocks().reshape(c.ny, c.nx, -1)
        dev = np.stack([allb[i, j] for i, j in offs])
        del allb, op
    else:
        dev = None
    tdev = time.time() - t0
    dw = [emie.design_offset_filters(i, j, c.hx, c.hy) for i, j in offs]
    hxn = np.nextafter(c.hx, np.inf)
    hyn = np.nextafter(c.hy, np.inf)
    base = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, c.hy, c.omega)
    cx = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, hxn, c.hy, c.omega)
    cy = R.RefCase(c.tops, c.sigma, c.breaks, c.nx, c.ny, c.hx, hyn, c.omega)

    def one(idx):
        i, j = offs[idx]
        return (base.block(i, j), cx.block(i, j), cy.block(i, j), base.block_weights(i, j, dw[idx][0], dw[idx][1]))

    t0 = time.time()
    with ThreadPoolExecutor(32) as ex:
        res = list(ex.map(one, range(len(offs))))
    tref = time.time() - t0
    ref = np.stack([r[0] for r in res])
    refx = np.stack([r[1] for r in res])
    refy = np.stack([r[2] for r in res])
    refw = np.stack([r[3] for r in res])
    out = ROOT / "gpurun_out" / f"greens_probe_cfg{k}.npz"
    out.parent.mkdir(exist_ok=True)
    np.savez_compressed(out, offs=np.array(offs), dev=dev if dev is not None else np.zeros(0), ref=ref, refx=refx,
                        refy=refy, refw=refw, devw=np.stack([w for w, _ in dw]))
    scale = np.max(np.abs(ref), axis=1)
    sens = np.maximum(np.max(np.abs(refx - ref), axis=1), np.max(np.abs(refy - ref), axis=1)) / scale
    efil = np.max(np.abs(refw - ref), axis=1) / scale
    line = f"cfg{k}: {len(offs)} offsets, device build {tdev:.1f} s, reference {tref:.1f} s\n"
    line += f"  1-ulp sensitivity   max {sens.max():.2e} median {np.median(sens):.2e}\n"
    line += f"  filter design part  max {efil.max():.2e} median {np.median(efil):.2e}  ratio-to-sens max {np.max(efil / sens):.2f}\n"
    if dev is not None:
        edev = np.max(np.abs(dev - ref), axis=1) / scale
        eacc = np.max(np.abs(dev - refw), axis=1) / scale
        line += f"  device total        max {edev.max():.2e} median {np.median(edev):.2e}  ratio-to-sens max {np.max(edev / sens):.2f} median {np.median(edev / sens):.2f}\n"
        line += f"  accumulation part   max {eacc.max():.2e} median {np.median(eacc):.2e}  ratio-to-sens max {np.max(eacc / sens):.2f}\n"
        worst = np.argsort(-(edev / sens))[:5]
        for w in worst:
            line += f"    offset {offs[w]}: dev {edev[w]:.2e} sens {sens[w]:.2e} filt {efil[w]:.2e} acc {eacc[w]:.2e}\n"
    print(line, flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:] or ["1"]:
        run(int(a))
