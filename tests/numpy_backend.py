"""NumpyBackend: the sharded apply's stages (lateral transforms, mode
contraction, column moves) restated with numpy over oracle/emie_oracle.py —
TEST INFRASTRUCTURE ONLY, the host backend of the gloo CPU tests of the
exchange logic in paper_1512_06126_b200/distributed.py (the product path is
distributed.CudaBackend)."""
from __future__ import annotations

import numpy as np

from paper_1512_06126_b200.distributed import ShardPlan, mirror_modes


class NumpyBackend:
    """The same stages restated with numpy (oracle/emie_oracle.py): test
    infrastructure for the gloo CPU tests of the exchange logic."""

    def __init__(self, plan: ShardPlan, rank: int, comp, dims, diag_slab, xp=None):
        import torch
        self.torch = torch
        self.plan, self.rank, self.comp, self.dims = plan, rank, comp, dims
        self.s, self.r1, self.r2 = (np.asarray(d) for d in diag_slab)
        self._orc = None

    def _oracle(self):
        if self._orc is None:
            import emie_oracle  # tests put oracle/ on sys.path
            self._orc = emie_oracle
        return self._orc

    def empty(self, shape):
        return self.torch.empty(shape, dtype=self.torch.complex128)

    def zeros(self, shape):
        return self.torch.zeros(shape, dtype=self.torch.complex128)

    def lateral_forward(self, U, nrhs):
        P = self.plan
        nzl = P.nzl(self.rank)
        u = U.numpy().reshape(nrhs, 3, nzl * P.ny * P.nx) * self.r2[None, None, :]
        u = u.reshape(nrhs, 3 * nzl, P.ny, P.nx)
        pad = np.zeros((nrhs, 3 * nzl, P.ey, P.ex), np.complex128)
        pad[:, :, :P.ny, :P.nx] = u
        F = np.fft.fft2(pad, axes=(2, 3))  # [r][plane][my][mx]
        S = np.ascontiguousarray(F.transpose(0, 3, 2, 1)).reshape(nrhs, P.E, 3 * nzl)  # m = mx*ey + my
        return self.torch.from_numpy(S)

    def lateral_forward_into(self, U, S, nrhs):
        S.copy_(self.lateral_forward(U, nrhs))

    def contract(self, S, nrhs, q0, q1):
        P = self.plan
        O = self._oracle()
        Sn = S.numpy()
        # the rank's quadrant modes (octant plans: its rows' modes and their transposes)
        qms = P.qmodes[self.rank] if (q0, q1) == (P.q[self.rank], P.q[self.rank + 1]) else range(q0, q1)
        for qm in qms:
            for m in mirror_modes(qm, P.qx, P.ex, P.ey):
                mx, my = divmod(m, P.ey)
                M = O._mode_matrix(self.comp, self.dims, P.nz, my, mx)
                for r in range(nrhs):
                    Sn[r, m] = M @ Sn[r, m]

    def lateral_inverse(self, S, U, nrhs):
        P = self.plan
        nzl = P.nzl(self.rank)
        F = S.numpy().reshape(nrhs, P.ex, P.ey, 3 * nzl).transpose(0, 3, 2, 1)
        b = np.fft.ifft2(F, axes=(2, 3))[:, :, :P.ny, :P.nx].reshape(nrhs, 3, -1)
        u = U.numpy().reshape(nrhs, 3, -1)
        out = self.s[None, None, :] * u + self.r1[None, None, :] * b
        return self.torch.from_numpy(np.ascontiguousarray(out).reshape(U.shape))

    def move(self, src, dst, nrhs, g, E, sdesc, ddesc, nzh):
        idx = self.plan.modes[g]
        s_arr, d_arr = src.numpy().reshape(-1), dst.numpy().reshape(-1)
        ni = len(idx)
        r = np.arange(nrhs)[:, None, None, None]
        i = np.arange(ni)[None, :, None, None]
        c = np.arange(3)[None, None, :, None]
        z = np.arange(nzh)[None, None, None, :]
        ms = r * E + idx[i] if sdesc[0] else r * ni + i
        md = r * E + idx[i] if ddesc[0] else r * ni + i
        d_arr[md * ddesc[1] + c * ddesc[2] + ddesc[3] + z] = s_arr[ms * sdesc[1] + c * sdesc[2] + sdesc[3] + z]
