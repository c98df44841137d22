"""Check the x<->y mirror symmetry of device-built Green blocks on square grids with hx = hy:
block (oi,oj) vs (oj,oi) with xx<->yy, xz<->yz (relative to the block max)."""
import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1512_06126_b200 as emie
from paper_1512_06126_b200 import configs
for k in (1, 2):
    cfg = configs.config(k)
    model = emie.LayeredModel(cfg.tops, cfg.sigma)
    grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
    sop = emie.assemble_operator(grid, model, cfg.omega, keep_blocks=True)
    b = sop.blocks()  # (ny, nx, nent)
    nz = cfg.nz; nt = nz*(nz+1)//2; nf = nz*nz
    xx = b[..., :nt]; yy = b[..., nt:2*nt]; zz = b[..., 2*nt:3*nt]; xy = b[..., 3*nt:4*nt]
    xz = b[..., 4*nt:4*nt+nf]; yz = b[..., 4*nt+nf:]
    T = lambda a: np.swapaxes(a, 0, 1)
    def rel(a, c):
        num = np.max(np.abs(a - c), axis=-1); den = np.max(np.abs(b), axis=-1)
        return float(np.max(num / den))
    print(f"cfg{k}: xx~yy^T {rel(xx, T(yy)):.2e}  zz~zz^T {rel(zz, T(zz)):.2e}  xy~xy^T {rel(xy, T(xy)):.2e}  xz~yz^T {rel(xz, T(yz)):.2e}  xz vs xz^T {rel(xz, T(xz)):.2e}")
