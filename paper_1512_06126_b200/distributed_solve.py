"""FGMRES on depth-sharded vectors.

The reference's restarted FGMRES (src/cie.cpp:117-238) with the operator
apply sharded as in distributed.py: every rank holds the depth slab of every
Krylov vector, runs the vector kernels on it and all-reduces the local sums
(2(j+1)+1 doubles per CGS2 pass, one norm per step), so all ranks carry the
same Hessenberg matrix, rotations and decisions. The orthogonalisation is the
CGS2 of the single-GPU solver (solver.cu: dots; update fused with the second
pass's dots; update with the new norm), the host arithmetic is
fgmres_device's, step for step.

Plumbing only: the vector kernels are the library's (emie_cu_vec_*, the tiled
CGS2 sweeps) on this rank's slab; the reductions are torch.distributed
all-reduces (NCCL between GPUs) or, for G virtual ranks in one process (the
one-GPU tests), sums over the ranks in rank order. A NumPy slab backend runs
the same solver in the gloo CPU tests.
"""
from __future__ import annotations

import ctypes
import math
from typing import Callable, List, Sequence

import numpy as np


# --------------------------------------------------------- slab vectors ----
class CudaSlabOps:
    """One rank's slab vector kernels through the C ABI (torch complex128
    CUDA tensors; reductions come back as float64 CUDA tensors)."""

    def __init__(self):
        import torch
        from . import lib, _check
        self.torch, self.L, self._check = torch, lib(), _check

    def _st(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    @staticmethod
    def _p(t):
        return ctypes.c_void_p(t.data_ptr())

    def zeros(self, shape):
        return self.torch.zeros(shape, dtype=self.torch.complex128, device="cuda")

    def reals(self, k):
        return self.torch.empty(k, dtype=self.torch.float64, device="cuda")

    def dots(self, V, nv, w, with_norm):
        out = self.reals(2 * nv + 1)
        n = w.numel()
        self._check(self.L.emie_cu_vec_dots(self._p(V), ctypes.c_longlong(V.shape[1]), nv, self._p(w),
                                            ctypes.c_longlong(n), int(with_norm), self._p(out), self._st()))
        return out

    def update(self, w, V, nv, h, want):
        """w -= V h; then the new w's dots against V ("dots") or |w|^2 ("norm")."""
        out = self.reals(2 * nv if want == "dots" else 1)
        d = self._p(out) if want == "dots" else None
        q = self._p(out) if want == "norm" else None
        self._check(self.L.emie_cu_vec_update(self._p(w), self._p(V), ctypes.c_longlong(V.shape[1]), nv,
                                              self._p(h), ctypes.c_longlong(w.numel()), d, q, self._st()))
        return out

    def combine(self, x, V, nv, y):
        self._check(self.L.emie_cu_vec_combine(self._p(x), self._p(V), ctypes.c_longlong(V.shape[1]), nv,
                                               self._p(y), ctypes.c_longlong(x.numel()), self._st()))

    def scale(self, y, x, a):
        self._check(self.L.emie_cu_vec_scale(self._p(y), self._p(x), ctypes.c_double(a),
                                             ctypes.c_longlong(x.numel()), self._st()))

    def residual(self, r, b, t):
        out = self.reals(1)
        self._check(self.L.emie_cu_vec_residual(self._p(r), self._p(b), self._p(t), ctypes.c_longlong(r.numel()),
                                                self._p(out), self._st()))
        return out

    def upload(self, vals):
        return self.torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64)).cuda()


class NumpySlabOps:
    """The same operations on CPU tensors with numpy (test infrastructure:
    the gloo tests of the sharded solver's host logic)."""

    def __init__(self):
        import torch
        self.torch = torch

    def zeros(self, shape):
        return self.torch.zeros(shape, dtype=self.torch.complex128)

    def reals(self, k):
        return self.torch.zeros(k, dtype=self.torch.float64)

    def dots(self, V, nv, w, with_norm):
        Vn, wn = V.numpy()[:nv], w.numpy().reshape(-1)
        d = np.conj(Vn) @ wn if nv else np.zeros(0, np.complex128)
        out = np.zeros(2 * nv + 1)
        out[0:2 * nv:2], out[1:2 * nv:2] = d.real, d.imag
        out[2 * nv] = np.vdot(wn, wn).real if with_norm else 0.0
        return self.torch.from_numpy(out)

    def update(self, w, V, nv, h, want):
        hn = h.numpy()
        hc = hn[0:2 * nv:2] + 1j * hn[1:2 * nv:2]
        wn = w.numpy().reshape(-1)
        Vn = V.numpy()[:nv]
        for l in range(nv):
            wn -= hc[l] * Vn[l]
        if want == "dots":
            d = np.conj(Vn) @ wn
            out = np.zeros(2 * nv)
            out[0::2], out[1::2] = d.real, d.imag
        else:
            out = np.array([np.vdot(wn, wn).real])
        return self.torch.from_numpy(out)

    def combine(self, x, V, nv, y):
        yn = y.numpy()
        xn = x.numpy().reshape(-1)
        for k in range(nv):
            xn += (yn[2 * k] + 1j * yn[2 * k + 1]) * V.numpy()[k]

    def scale(self, y, x, a):
        y.numpy().reshape(-1)[:] = a * x.numpy().reshape(-1)

    def residual(self, r, b, t):
        rn = r.numpy().reshape(-1)
        rn[:] = b.numpy().reshape(-1) - t.numpy().reshape(-1)
        return self.torch.from_numpy(np.array([np.vdot(rn, rn).real]))

    def upload(self, vals):
        return self.torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64))


# ------------------------------------------------------------ reducers ----
class LoopbackReducer:
    """G virtual ranks in one process: the all-reduce is a sum over the
    per-rank arrays in rank order; every rank gets the sum back."""

    def __call__(self, parts: Sequence) -> tuple:
        host = [p.cpu().numpy() for p in parts]
        tot = host[0].copy()
        for h in host[1:]:
            tot = tot + h
        return tot


class TorchReducer:
    """One rank per process: torch.distributed all-reduce (sum) of the
    rank's local sums (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        self.group = group

    def __call__(self, parts: Sequence) -> np.ndarray:
        import torch.distributed as dist
        (t,) = parts
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()


# ------------------------------------------------------------ the solve ----
def _rotation(f: complex, g: complex):
    """make_rotation (cie.cpp:100-113): complex Givens with real cosine."""
    if g == 0:
        return 1.0, 0j
    if f == 0:
        return 0.0, np.conj(g) / abs(g)
    t = math.sqrt(abs(f) ** 2 + abs(g) ** 2)
    return abs(f) / t, f / abs(f) * np.conj(g) / t


def fgmres_sharded(apply: Callable[[List], List], ops: Sequence, reduce: Callable, rhs: Sequence,
                   tol: float = 1e-8, restart: int = 40, max_iters: int = 500):
    """FGMRES (cie.cpp:117-238) for nrhs right-hand sides in lockstep.

    apply(list of per-rank U (nrhs, n_local)) -> list of per-rank A U;
    ops: per-rank slab vector backends (CudaSlabOps / NumpySlabOps);
    reduce(list of per-rank local sums) -> the global sums (host numpy);
    rhs: per-rank (nrhs, n_local) slabs. Returns (per-rank x slabs, reports)."""
    from . import SolveReport
    if not (tol > 0.0) or restart < 1 or max_iters < 1:
        from . import InvalidArgument
        raise InvalidArgument("fgmres: bad solver configuration")
    G = len(ops)
    nrhs, n = rhs[0].shape[0], [b.shape[1] for b in rhs]
    m = restart
    V = [[ops[g].zeros((m + 1, n[g])) for g in range(G)] for _ in range(nrhs)]
    x = [ops[g].zeros((nrhs, n[g])) for g in range(G)]
    r = [ops[g].zeros((nrhs, n[g])) for g in range(G)]

    def red(fn):  # per-rank local sums -> global host values + per-rank device copies
        tot = reduce([fn(g) for g in range(G)])
        return tot, [ops[g].upload(tot) for g in range(G)]

    st = []
    for i in range(nrhs):
        bn2, _ = red(lambda g: ops[g].dots(V[i][g], 0, rhs[g][i], True))
        st.append(dict(bnorm=math.sqrt(bn2[0]), rnorm=0.0, iter=0, broke=False, phase="cycle",
                       status="max_iterations", history=[]))
        if st[i]["bnorm"] == 0.0:  # cie.cpp:124-128
            st[i].update(status="converged", phase="done")
            continue
        for g in range(G):
            r[g][i].copy_(rhs[g][i])
        st[i]["rnorm"] = st[i]["bnorm"]

    def start_cycle(i):
        s = st[i]
        if not s["iter"] < max_iters:
            return False
        for g in range(G):
            ops[g].scale(V[i][g][0], r[g][i], 1.0 / s["rnorm"])
        s.update(h=np.zeros((m, m + 1), np.complex128), c=np.zeros(m), sn=np.zeros(m, np.complex128),
                 gv=np.zeros(m + 1, np.complex128), cols=0, j=0, phase="inner")
        s["gv"][0] = s["rnorm"]
        return True

    for i in range(nrhs):
        if st[i]["phase"] == "cycle" and not start_cycle(i):
            st[i]["phase"] = "done"

    def close_cycle(i):
        s = st[i]
        cols = s["cols"]
        if cols > 0:  # back substitution (cie.cpp:205-215)
            y = np.zeros(cols, np.complex128)
            for k in range(cols - 1, -1, -1):
                acc = s["gv"][k]
                for l in range(k + 1, cols):
                    acc -= s["h"][l, k] * y[l]
                y[k] = acc / s["h"][k, k]
            yv = np.zeros(2 * cols)
            yv[0::2], yv[1::2] = y.real, y.imag
            for g in range(G):
                ops[g].combine(x[g][i], V[i][g], cols, ops[g].upload(yv))
        s["phase"] = "residual"

    while True:
        active = [i for i in range(nrhs) if st[i]["phase"] in ("inner", "residual")]
        if not active:
            break
        # one batched (all rhs) sharded apply per round
        U = [ops[g].zeros((nrhs, n[g])) for g in range(G)]
        for i in active:
            for g in range(G):
                U[g][i].copy_(V[i][g][st[i]["j"]] if st[i]["phase"] == "inner" else x[g][i])
        W = apply(U)
        for i in active:
            s = st[i]
            w = [W[g][i] for g in range(G)]
            if s["phase"] == "residual":  # cie.cpp:217-229
                rr, _ = red(lambda g: ops[g].residual(r[g][i], rhs[g][i], w[g]))
                s["rnorm"] = math.sqrt(rr[0])
                if s["rnorm"] / s["bnorm"] <= tol:
                    s.update(status="converged", phase="done")
                elif s["broke"]:
                    s.update(status="breakdown", phase="done")
                elif not start_cycle(i):
                    s["phase"] = "done"
                continue
            j = s["j"]
            nv = j + 1
            d1, h1 = red(lambda g: ops[g].dots(V[i][g], nv, w[g], True))
            d2, h2 = red(lambda g: ops[g].update(w[g], V[i][g], nv, h1[g], "dots"))
            nn, _ = red(lambda g: ops[g].update(w[g], V[i][g], nv, h2[g], "norm"))
            s["iter"] += 1
            hj = s["h"][j]
            wn0 = math.sqrt(d1[2 * nv])
            hj[:nv] += d1[0:2 * nv:2] + 1j * d1[1:2 * nv:2]
            hj[:nv] += d2[0::2] + 1j * d2[1::2]
            hnext = math.sqrt(nn[0])
            for k in range(j):
                t = s["c"][k] * hj[k] + s["sn"][k] * hj[k + 1]
                hj[k + 1] = -np.conj(s["sn"][k]) * hj[k] + s["c"][k] * hj[k + 1]
                hj[k] = t
            end = False
            if hnext <= 1e-13 * max(wn0, 1e-300):  # breakdown test (cie.cpp:171-187)
                colmax = max([hnext] + [abs(v) for v in hj[:nv]])
                if abs(hj[j]) > 1e-13 * max(colmax, 1e-300):
                    s["cols"] = nv
                else:
                    s["cols"] = j
                    s["broke"] = True
                    s["history"].append(s["rnorm"] / s["bnorm"])
                end = True
            else:
                hj[j + 1] = hnext
                for g in range(G):
                    ops[g].scale(V[i][g][j + 1], w[g], 1.0 / hnext)
                c, sn = _rotation(hj[j], hnext)
                s["c"][j], s["sn"][j] = c, sn
                t = c * hj[j] + sn * hj[j + 1]
                hj[j + 1] = 0.0
                hj[j] = t
                s["gv"][j + 1] = -np.conj(sn) * s["gv"][j]
                s["gv"][j] = c * s["gv"][j]
                s["cols"] = nv
                est = abs(s["gv"][j + 1]) / s["bnorm"]
                s["history"].append(est)
                if est <= tol:
                    end = True
            if not end:
                s["j"] += 1
                if not (s["j"] < m and s["iter"] < max_iters):
                    end = True
            if end:
                close_cycle(i)
    reports = [SolveReport(s["status"], s["iter"], 0.0 if s["bnorm"] == 0.0 else s["rnorm"] / s["bnorm"],
                           list(s["history"])) for s in st]
    return x, reports
