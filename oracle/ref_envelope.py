"""The reference's own arithmetic envelope of its Green's blocks — TEST
INFRASTRUCTURE ONLY (tests/test_gpu_greens_parity.py, tools/).

The reference's compressed blocks (assemble_block, src/greens.cpp:150-221)
are determined only to the accuracy its own floating-point evaluation
allows: the lateral filter sums are ill-conditioned (V1 + V3 cancels up to 13
digits as lambda -> 0 and V2 + V5 as lambda -> inf, layered.cpp:397-408 with
the W11d/W20d forms of layered.cpp:305-315; the filter design deconvolves by
an input spectrum floored at 1e-12 of its maximum, hankel.cpp:229-231). This
module measures how far the reference moves under changes that leave the
algorithm and the IEEE double arithmetic intact:

  hx+ / hy+  the cell size moved by one ulp (nextafter), the sensitivity to
             its inputs;
  fma        the same sources compiled with FMA contraction
             (oracle/_ref_fma: -mfma -ffp-contract=fast, what every GPU
             compiler does by default), the sensitivity to legitimate
             rounding choices.

Each variant runs in its own process (the two builds of libemie_ref.so must
not share one address space). CLI (used by reference_blocks):

    python oracle/ref_envelope.py CASE.npz OUT.npz VARIANT
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def _blocks_here(case: dict, variant: str) -> dict:
    sys.path.insert(0, str(HERE))
    import ref_binding as R
    offs = case["offs"]
    args = (case["tops"], case["sigma"], case["breaks"], int(case["nx"]), int(case["ny"]))
    hx, hy, om = float(case["hx"]), float(case["hy"]), float(case["omega"])
    cases = {"base": R.RefCase(*args, hx, hy, om)}
    if variant == "_ref":
        cases["hx+"] = R.RefCase(*args, np.nextafter(hx, np.inf), hy, om)
        cases["hy+"] = R.RefCase(*args, hx, np.nextafter(hy, np.inf), om)
    jobs = [(name, i) for name in cases for i in range(len(offs))]

    def one(job):
        name, i = job
        return cases[name].block(int(offs[i][0]), int(offs[i][1]))

    with ThreadPoolExecutor(min(64, os.cpu_count() or 8)) as ex:
        res = list(ex.map(one, jobs))
    out = {}
    for name in cases:
        out[name] = np.stack([r for (n, _), r in zip(jobs, res) if n == name])
    return out


def reference_blocks(tops, sigma, breaks, nx, ny, hx, hy, omega, offs) -> dict:
    """Blocks of the reference at the signed offsets offs (n, 2) ->
    {"ref", "hx+", "hy+", "fma"} each (n, 2nz(2nz+1)), in two child processes."""
    with tempfile.TemporaryDirectory() as d:
        cpath = Path(d) / "case.npz"
        np.savez(cpath, tops=np.asarray(tops, np.float64), sigma=np.asarray(sigma, np.complex128),
                 breaks=np.asarray(breaks, np.float64), nx=nx, ny=ny, hx=hx, hy=hy, omega=omega,
                 offs=np.asarray(offs, np.int64).reshape(-1, 2))
        procs = []
        for v in ("_ref", "_ref_fma"):
            env = dict(os.environ, EMIE_REF_VARIANT=v)
            procs.append((v, subprocess.Popen([sys.executable, str(Path(__file__)), str(cpath),
                                               str(Path(d) / f"{v}.npz"), v], env=env,
                                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        for v, p in procs:
            out, _ = p.communicate(timeout=3600)
            if p.returncode != 0:
                raise RuntimeError(f"reference variant {v} failed:\n{out.decode()}")
        a = dict(np.load(Path(d) / "_ref.npz"))
        b = dict(np.load(Path(d) / "_ref_fma.npz"))
    return {"ref": a["base"], "hx+": a["hx+"], "hy+": a["hy+"], "fma": b["base"]}


def _chain_here(case: dict) -> dict:
    """The reference pipeline of one case: assemble_operator +
    transform_operator + build_system (ref_build), then solve_cie for each
    right-hand side (cie.cpp:240-249)."""
    sys.path.insert(0, str(HERE))
    import ref_binding as R
    c = R.RefCase(case["tops"], case["sigma"], case["breaks"], int(case["nx"]), int(case["ny"]), float(case["hx"]),
                  float(case["hy"]), float(case["omega"]), case["sigma_a"])
    blocks, _, _ = c.build()
    xs, its = [], []
    for b in case["rhs"]:
        x, rep = c.solve(b, float(case["tol"]), int(case["restart"]), int(case["max_iters"]))
        xs.append(x)
        its.append(rep["iterations"])
    out = {"x": np.stack(xs), "iters": np.array(its)}
    if int(case["want_blocks"]):
        out["blocks"] = blocks
    return out


def reference_chain(tops, sigma, breaks, nx, ny, hx, hy, omega, sigma_a, rhs, tol, restart=40, max_iters=500,
                    variants=("_ref", "_ref_fma"), want_blocks=False) -> dict:
    """{variant: {"x": solutions (nrhs, n), "iters": (nrhs,)[, "blocks"]}} of
    the reference's own build + solve, one child process per variant."""
    with tempfile.TemporaryDirectory() as d:
        cpath = Path(d) / "case.npz"
        np.savez(cpath, tops=np.asarray(tops, np.float64), sigma=np.asarray(sigma, np.complex128),
                 breaks=np.asarray(breaks, np.float64), nx=nx, ny=ny, hx=hx, hy=hy, omega=omega,
                 sigma_a=np.asarray(sigma_a, np.complex128).reshape(-1), rhs=np.asarray(rhs, np.complex128),
                 tol=tol, restart=restart, max_iters=max_iters, want_blocks=int(want_blocks))
        procs = []
        for v in variants:
            env = dict(os.environ, EMIE_REF_VARIANT=v)
            procs.append((v, subprocess.Popen([sys.executable, str(Path(__file__)), str(cpath),
                                               str(Path(d) / f"{v}.npz"), "chain"], env=env,
                                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        res = {}
        for v, p in procs:
            out, _ = p.communicate(timeout=7200)
            if p.returncode != 0:
                raise RuntimeError(f"reference variant {v} failed:\n{out.decode()}")
            res[v] = dict(np.load(Path(d) / f"{v}.npz"))
    return res


def envelope(blocks: dict) -> np.ndarray:
    """Per-block envelope: the largest move of the reference under the
    variants, relative to the block's max modulus."""
    ref = blocks["ref"]
    scale = np.max(np.abs(ref), axis=1)
    moves = [np.max(np.abs(blocks[k] - ref), axis=1) for k in ("hx+", "hy+", "fma")]
    return np.max(moves, axis=0) / scale


if __name__ == "__main__":
    case = dict(np.load(sys.argv[1]))
    res = _chain_here(case) if sys.argv[3] == "chain" else _blocks_here(case, sys.argv[3])
    np.savez(sys.argv[2], **res)
