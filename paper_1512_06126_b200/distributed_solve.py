"""FGMRES on depth-sharded vectors.

The reference's restarted FGMRES (src/cie.cpp:117-238) with the operator
apply sharded as in distributed.py: every rank holds the depth slab of every
Krylov vector, runs the vector kernels on it and all-reduces the local sums
(2(j+1)+1 doubles per CGS2 pass, one norm per step), so all ranks carry the
same Hessenberg matrix, rotations and decisions. The orthogonalisation is
the single-GPU solver's (solver.cu): DCGS2 by default -- one dots sweep
giving both V^H w and v_j's delayed reorthogonalisation dots, one update
sweep correcting v_j in place and projecting w, so two all-reduces per step
(4nv + 1 doubles) -- or CGS2 (three sweeps, three all-reduces); the host
arithmetic is fgmres_device's, step for step.

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

    def dcgs_dots(self, V, nv, w):
        out = self.reals(4 * nv)
        self._check(self.L.emie_cu_vec_dcgs_dots(self._p(V), ctypes.c_longlong(V.shape[1]), nv, self._p(w),
                                                 ctypes.c_longlong(w.numel()), self._p(out), self._st()))
        return out

    def dcgs_update(self, w, V, nv, coef):
        out = self.reals(1)
        self._check(self.L.emie_cu_vec_dcgs_update(self._p(w), self._p(V), ctypes.c_longlong(V.shape[1]), nv,
                                                   self._p(coef), ctypes.c_longlong(w.numel()), self._p(out),
                                                   self._st()))
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

    def dcgs_dots(self, V, nv, w):
        Vn, wn = V.numpy()[:nv], w.numpy().reshape(-1)
        out = np.zeros(4 * nv)
        d = np.conj(Vn) @ wn
        out[0:2 * nv:2], out[1:2 * nv:2] = d.real, d.imag
        out[2 * nv] = np.vdot(wn, wn).real
        a = np.conj(Vn[:nv - 1]) @ Vn[nv - 1]
        out[2 * nv + 1:4 * nv - 1:2], out[2 * nv + 2:4 * nv - 1:2] = a.real, a.imag
        out[4 * nv - 1] = np.vdot(Vn[nv - 1], Vn[nv - 1]).real
        return self.torch.from_numpy(out)

    def dcgs_update(self, w, V, nv, coef):
        c = coef.numpy()
        h = c[0:2 * nv:2] + 1j * c[1:2 * nv:2]
        a = c[2 * nv:4 * nv - 2:2] + 1j * c[2 * nv + 1:4 * nv - 2:2]
        Vn, wn = V.numpy(), w.numpy().reshape(-1)
        vj = Vn[nv - 1].copy()
        for l in range(nv - 1):
            vj -= a[l] * Vn[l]
        vj *= c[4 * nv - 2]
        Vn[nv - 1] = vj
        for l in range(nv - 1):
            wn -= h[l] * Vn[l]
        wn -= h[nv - 1] * vj
        return self.torch.from_numpy(np.array([np.vdot(wn, wn).real]))

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


def dcgs_coefficients(d: np.ndarray, nv: int):
    """DCGS2 step coefficients from the global dcgs_dots sums d (4nv values,
    the layout of solver.cu's MODE 3 / dcgs_coef_kernel): v_j's correction a
    (nv-1 complex), alpha = sqrt(|v_j|^2 - |a|^2), w's coefficients h against
    the corrected basis -> (coef [h][a][1/alpha] as float64, h, a, alpha)."""
    b = d[0:2 * nv:2] + 1j * d[1:2 * nv:2]
    a = d[2 * nv + 1:4 * nv - 1:2] + 1j * d[2 * nv + 2:4 * nv - 1:2]
    a2 = d[4 * nv - 1] - float(np.sum(a.real ** 2 + a.imag ** 2))
    alpha = math.sqrt(a2) if a2 > 0.0 else 0.0
    ia = 1.0 / alpha if alpha > 0.0 else 0.0
    h = b.copy()
    h[nv - 1] = (b[nv - 1] - np.sum(np.conj(a) * b[:nv - 1])) * ia
    coef = np.zeros(4 * nv - 1)
    coef[0:2 * nv:2], coef[1:2 * nv:2] = h.real, h.imag
    coef[2 * nv:4 * nv - 2:2], coef[2 * nv + 1:4 * nv - 2:2] = a.real, a.imag
    coef[4 * nv - 2] = ia
    return coef, h, a, alpha


def fgmres_sharded(apply: Callable[[List], List], ops: Sequence, reduce: Callable, rhs: Sequence,
                   tol: float = 1e-8, restart: int = 40, max_iters: int = 500, ortho: str = "dcgs2"):
    """FGMRES (cie.cpp:117-238) for nrhs right-hand sides in lockstep.

    apply(list of per-rank U (nrhs, n_local)) -> list of per-rank A U;
    ops: per-rank slab vector backends (CudaSlabOps / NumpySlabOps);
    reduce(list of per-rank local sums) -> the global sums (host numpy);
    rhs: per-rank (nrhs, n_local) slabs. Returns (per-rank x slabs, reports).
    ortho: "dcgs2" (the single-GPU solver's default: one dots sweep and one
    update sweep per step, two all-reduces) or "cgs2" (three sweeps, three
    all-reduces); restarts above 40 use CGS2."""
    from . import SolveReport
    if not (tol > 0.0) or restart < 1 or max_iters < 1:
        from . import InvalidArgument
        raise InvalidArgument("fgmres: bad solver configuration")
    G = len(ops)
    nrhs, n = rhs[0].shape[0], [b.shape[1] for b in rhs]
    m = restart
    dcgs = ortho == "dcgs2" and m + 1 <= 41
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
                 gv=np.zeros(m + 1, np.complex128), cols=0, j=0, phase="inner",
                 hraw=np.zeros((m, m + 1), np.complex128), gpre=np.zeros(m + 1, np.complex128),
                 acoef=np.zeros((m + 1, m + 1), np.complex128), rho=np.zeros(m + 1), alpha=np.ones(m + 1))
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
            if dcgs:  # the applies saw v_j before its correction: v_j(applied) = alpha_j v_j + V a_j
                y = np.array([s["alpha"][k] * y[k] + np.sum(s["acoef"][k + 1:cols, k] * y[k + 1:cols])
                              for k in range(cols)])
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
            hj = s["h"][j]
            if dcgs:
                d, _ = red(lambda g: ops[g].dcgs_dots(V[i][g], nv, w[g]))
                coef, hc, acol, alpha = dcgs_coefficients(d, nv)
                nn, _ = red(lambda g: ops[g].dcgs_update(w[g], V[i][g], nv, ops[g].upload(coef)))
                s["iter"] += 1
                wn0 = math.sqrt(d[2 * nv])
                hnext = math.sqrt(nn[0])
                s["alpha"][j] = alpha
                s["acoef"][j, :j] = acol
                if j >= 1:  # column j-1 gains rho_{j-1} a, subdiagonal rho_{j-1} alpha; re-rotated
                    hr = s["hraw"][j - 1]
                    hr[:j] += s["rho"][j - 1] * acol
                    hr[j] = s["rho"][j - 1] * alpha
                    hc1 = s["h"][j - 1]
                    hc1[:j + 1] = hr[:j + 1]
                    for k in range(j - 1):
                        t = s["c"][k] * hc1[k] + s["sn"][k] * hc1[k + 1]
                        hc1[k + 1] = -np.conj(s["sn"][k]) * hc1[k] + s["c"][k] * hc1[k + 1]
                        hc1[k] = t
                    c1, sn1 = _rotation(hc1[j - 1], hc1[j])
                    s["c"][j - 1], s["sn"][j - 1] = c1, sn1
                    t = c1 * hc1[j - 1] + sn1 * hc1[j]
                    hc1[j] = 0.0
                    hc1[j - 1] = t
                    s["gv"][j] = -np.conj(sn1) * s["gpre"][j - 1]
                    s["gv"][j - 1] = c1 * s["gpre"][j - 1]
                s["hraw"][j, :nv] = hc
                s["hraw"][j, nv] = hnext
                s["rho"][j] = hnext
                hj[:nv] = hc
            else:
                d1, h1 = red(lambda g: ops[g].dots(V[i][g], nv, w[g], True))
                d2, h2 = red(lambda g: ops[g].update(w[g], V[i][g], nv, h1[g], "dots"))
                nn, _ = red(lambda g: ops[g].update(w[g], V[i][g], nv, h2[g], "norm"))
                s["iter"] += 1
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
                s["gpre"][j] = s["gv"][j]
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
