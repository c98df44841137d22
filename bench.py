#!/usr/bin/env python
"""Benchmark of the CIE operator apply (BASELINE.json metric: "CIE operator
applies/s (complex128) at 128x128x32; Green's tensor build time").

Workload (config 3, the reference's headline single-GPU config): the
128x128x32 model of paper_1512_06126_b200/configs.py, 5-layer background,
seeded log10 sigma in [-4, 1], 1 Hz, both MT polarisations. One step is one
apply(SystemOperator) (include/emie/cie.hpp:39) on the two polarisations'
fields (nrhs = 2, as FGMRES runs them in lockstep), so one step = 2 applies.
The operator is built on the device by the Green's build (its wall time is
reported as greens_build_s, the second half of the metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): weak scaling over independent
frequencies (config 5's sweep): rank r owns frequency r, builds its own
operator and applies it; there is no data-path collective. value = all
ranks' applies / max-over-ranks device time.

--impl reference times the reference's own CPU implementation
(oracle/_ref, compiled from its sources) of the same apply on this host's
cores, same workload and metric; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CIE operator applies/s (complex128) at 128x128x32"  # config 3 (the default)


def metric_for(cfg):
    return f"CIE operator applies/s (complex128) at {cfg.nx}x{cfg.ny}x{cfg.nz}"
UNIT = "applies/s"
NRHS = 2
LIB_POOL_RESERVE = 8 << 30  # bytes reserved in the library's memory pool at init (a cfg3 build's workspaces: ~4 GB)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)  # 100 timed applies (SURVEY.md §8(d) timing protocol)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=20)
    p.add_argument("--no-solve", action="store_true", help="skip the FGMRES solve timing")
    p.add_argument("--strong", action="store_true",
                   help="strong scaling of one grid: depth-slab / mode-shard apply over the N ranks")
    p.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                   help="--strong: column transposes as peer stores (IPC buffers, flag barriers) or NCCL all-to-all")
    p.add_argument("--peer-sync", default="flags", choices=["flags", "host"],
                   help="--strong --exchange peer: device flag barriers, or stream sync + a host barrier (ranks "
                        "sharing one GPU: no kernel may spin on another process's flag)")
    p.add_argument("--shard-layout", default="auto", choices=["auto", "octant", "quadrant"],
                   help="--strong: octant rows per rank (square grids with hx == hy: each stored block read once "
                        "for a mode and its transpose) or quadrant-mode ranges; auto = octant where possible")
    p.add_argument("--check", action="store_true",
                   help="--strong: compare the sharded apply with the unsharded device apply (gathered on rank 0)")
    return p.parse_args()


def host_cpu():
    """Host cores for the CPU baselines (physical cores and the
    lscpu model name): logical CPUs, physical cores, model."""
    info = {"logical_cpus": os.cpu_count(), "physical_cores": None, "model": None}
    try:
        out = subprocess.run(["lscpu", "-p=CORE,SOCKET"], capture_output=True, text=True, timeout=10).stdout
        cores = {tuple(r.split(",")) for r in out.splitlines() if r and not r.startswith("#")}
        info["physical_cores"] = len(cores) or None
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.lower().startswith("model name"):
                info["model"] = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    info["threads_used"] = info["physical_cores"] or info["logical_cpus"]
    return info


def config_of(args, cfg, freq=None):
    """The workload dict both arms print (same keys and values)."""
    return {"workload": f"cfg{args.config} {cfg.nx}x{cfg.ny}x{cfg.nz} (5-layer background), "
                        "apply(SystemOperator) on both MT polarisations per step (nrhs=2)",
            "nrhs": NRHS, "frequency_hz": cfg.freqs[0] if freq is None else freq,
            "grid": [cfg.nx, cfg.ny, cfg.nz], "cell_m": [cfg.hx, cfg.hy],
            "l2": f"inputs larger than L2 (the {spectra_gb(cfg):.2f} GB operator spectra are read every step)"}


def spectra_gb(cfg):
    """Size of the reference's spectral operator (toeplitz.cpp:86-90): quadrant
    modes x 2nz(2nz+1) complex128."""
    q = lambda n: smooth_embedding(2 * n - 1) // 2 + 1  # noqa: E731
    return q(cfg.nx) * q(cfg.ny) * 2 * cfg.nz * (2 * cfg.nz + 1) * 16 / 1e9


def smooth_embedding(n):  # toeplitz.cpp:18-26 (2,3,5-smooth), for the label only
    m = max(1, n)
    while True:
        k = m
        for f in (2, 3, 5):
            while k % f == 0:
                k //= f
        if k == 1:
            return m
        m += 1


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=self.out, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.3)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.out.flush()
        rows = [r.split(",") for r in Path(self.out.name).read_text().strip().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, v in zip(names, r[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        os.unlink(self.out.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------ reference arm ----
def write_case(cfg, path, omega):
    import ref_binding as R
    R.write_case(path, cfg.tops, cfg.sigma, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy, omega,
                 cfg.sigma_a)


def reference_apply_rate(cfg, reps, threads=None):
    """The reference's apply(SystemOperator) (src/cie.cpp:56-73) timed on the
    host cores through oracle/_ref/emie_ref_tool (all OpenMP threads)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_binding as R
    if not R.TOOL.exists():
        R.build()
    with tempfile.TemporaryDirectory() as td:
        case = Path(td) / "case.bin"
        write_case(cfg, case, cfg.omega)
        out = R.run_tool("bench-apply", case, reps, NRHS, threads=threads)
    d = json.loads(out)
    return d


def reference_greens_seconds(cfg, stride=16, threads=None):
    """The reference's Green's build (assemble_block over the offsets with its
    per-thread designers and shared moment memo, greens.cpp:332-371) timed on
    every stride-th offset through oracle/_ref/emie_ref_tool and extrapolated
    linearly to all nx*ny offsets."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_binding as R
    if not R.TOOL.exists():
        R.build()
    with tempfile.TemporaryDirectory() as td:
        case = Path(td) / "case.bin"
        write_case(cfg, case, cfg.omega)
        d = json.loads(R.run_tool("bench-greens", case, stride, threads=threads))
    d["extrapolated_s"] = d["seconds"] * d["total_offsets"] / d["offsets"]
    d["stride"] = stride
    return d


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1512_06126_b200 import configs
    cfg = configs.config(args.config)
    cpu = host_cpu()
    threads = cpu["threads_used"]
    d = reference_apply_rate(cfg, args.warmup + args.steps, threads=threads)
    times = d["times"][args.warmup:]
    tot = float(np.sum(times))
    value = NRHS * len(times) / tot
    line = {
        "impl": "reference", "metric": metric_for(cfg), "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": "synthetic (seeded config conductivity field, seeded fields; the reference applies a "
                "synthetic operator of the same shape -- its apply cost does not depend on the values)",
        "config": config_of(args, cfg),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": d["threads"], "kind": "reference",
                         "host": cpu,
                         "sample": f"{len(times)} steps x {NRHS} applies at cfg{args.config} (reference "
                                   "apply(SystemOperator), OpenMP on the physical cores, FFTW-API shim: "
                                   "no libfftw3 on the host)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        g = reference_greens_seconds(cfg, 16, threads=threads)
        line["greens_build_s"] = g["extrapolated_s"]
        line["greens_sample"] = (f"assemble_block over every {g['stride']}th offset ({g['offsets']} of "
                                 f"{g['total_offsets']}, {g['seconds']:.2f} s on {g['threads']} threads), "
                                 "extrapolated linearly")
    except Exception as ex:  # noqa: BLE001
        line["greens_build_s"] = None
        line["greens_sample"] = f"unavailable: {ex}"
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- our arm ----
def run_ours(args):
    import ctypes

    import torch
    import paper_1512_06126_b200 as emie
    from paper_1512_06126_b200 import configs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # EMIE_BENCH_BACKEND=gloo: a CPU-side process group (a multi-rank dry run of
    # this script on fewer GPUs; ranks share devices, their work is independent)
    backend = os.environ.get("EMIE_BENCH_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    cfg = configs.config(args.config)
    freqs = configs.config(5).freqs
    from paper_1512_06126_b200.sharding import shard_indices
    # weak scaling over the config-5 sweep: rank r owns frequency r (round robin)
    freq = cfg.freqs[0] if world == 1 else freqs[shard_indices(len(freqs), world, rank)[0]]
    omega = 2.0 * np.pi * freq
    model = emie.LayeredModel(cfg.tops, cfg.sigma)
    grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
    grid.sigma_a[...] = cfg.sigma_a

    L = emie.lib()
    # library initialisation (CUDA loads kernels lazily, on first launch): one
    # tiny build + apply, and 8 GB reserved in the library's stream-ordered
    # memory pool (the device's first touch of fresh memory otherwise lands in
    # the first build: +15..300 ms, erratic), timed on its own as library_init_s
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    emie.warmup(reserve_bytes=LIB_POOL_RESERVE)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    # Green's build on the device (wall time, device synchronised): the first
    # build of this configuration in the process
    t0 = time.perf_counter()
    operator_src = "device Green's build"
    try:
        sop = emie.assemble_operator(grid, model, omega)
    except emie.EmieRuntimeError:
        operator_src = "synthetic compressed blocks (device Green's build unavailable)"
        rng = np.random.default_rng(5)
        nent = 2 * cfg.nz * (2 * cfg.nz + 1)
        blocks = (rng.standard_normal((cfg.ny, cfg.nx, nent)) +
                  1j * rng.standard_normal((cfg.ny, cfg.nx, nent))) * 1e-3
        sop = emie.transform_operator(blocks, cfg.nx, cfg.ny, cfg.nz, omega)
    torch.cuda.synchronize()
    greens_s = time.perf_counter() - t0
    # second build in the same process (allocator and modules warm; the first
    # operator released before, as a frequency sweep does, so its spectra
    # buffer is handed over instead of a fresh 1.1 GB cudaMalloc), with the
    # library's own CUDA-event stage timers: 5 = assemble kernel, 6 = spectra
    greens_warm_s, greens_stage = None, None
    if operator_src == "device Green's build":
        L.emie_cu_profile_enable.argtypes = [ctypes.c_int]
        L.emie_cu_profile_collect.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        ms8, cnt8 = np.zeros(8), np.zeros(8, np.int64)
        # median of three warm builds (host noise: one build of a run can take
        # several times the others)
        warm, stage_runs = [], []
        for _ in range(3):
            L.emie_cu_profile_collect(ms8.ctypes.data, cnt8.ctypes.data, 8)
            del sop
            torch.cuda.synchronize()
            L.emie_cu_profile_enable(1)
            t0 = time.perf_counter()
            sop = emie.assemble_operator(grid, model, omega)
            torch.cuda.synchronize()
            warm.append(time.perf_counter() - t0)
            L.emie_cu_profile_enable(0)
            L.emie_cu_profile_collect(ms8.ctypes.data, cnt8.ctypes.data, 8)
            stage_runs.append((float(ms8[5]), float(ms8[6])))
        i_med = int(np.argsort(warm)[1])
        greens_warm_s = warm[i_med]
        greens_stage = {"assemble_kernel_ms": round(stage_runs[i_med][0], 3),
                        "spectra_ms": round(stage_runs[i_med][1], 3),
                        "warm_builds_s": [round(w, 4) for w in warm]}
    system = emie.build_system(grid, sop)

    n = 3 * cfg.cells()
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    U = torch.complex(torch.rand(NRHS * n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1,
                      torch.rand(NRHS * n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1)
    W = torch.empty_like(U)
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)

    def step():
        emie._check(L.emie_cu_apply_system(system.handle, ctypes.c_void_p(U.data_ptr()),
                                           ctypes.c_void_p(W.data_ptr()), NRHS, sp))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    L.emie_cu_profile_enable.argtypes = [ctypes.c_int]
    L.emie_cu_profile_collect.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    L.emie_cu_probe_fp64.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]
    ms5 = np.zeros(5)
    cnt5 = np.zeros(5, np.int64)
    emie._check(L.emie_cu_profile_collect(ms5.ctypes.data, cnt5.ctypes.data, 5))  # drain
    emie._check(L.emie_cu_profile_enable(0))  # the timed loop runs uninstrumented
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.4)
    L.emie_cu_reset_launch_count()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record(stream)
    marks[0].record(stream)
    for i in range(args.steps):
        step()
        marks[i + 1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    per_step = np.array([marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)])
    if dist:
        dist.barrier()
    launches = int(L.emie_cu_launch_count())
    clk = clocks.stop()
    # stage breakdown (and the contraction time of the roofline) from a
    # separate instrumented pass: the library's per-stage CUDA events cost ~5 %
    # of the step, so they stay out of the timed loop
    emie._check(L.emie_cu_profile_enable(1))
    nprof = max(3, min(args.steps, 10))
    for _ in range(nprof):
        step()
    torch.cuda.synchronize()
    emie._check(L.emie_cu_profile_enable(0))
    emie._check(L.emie_cu_profile_collect(ms5.ctypes.data, cnt5.ctypes.data, 5))
    ms = e0.elapsed_time(e1)
    tmax = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if dist:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    value = world * NRHS * args.steps / (ms_max * 1e-3)

    # end to end through the reference-facing host-buffer C-ABI call
    # (--e2e-steps 0 skips it, e.g. for a launch-list capture of the device steps).
    # Headline: the K steps' fields (K x 2 polarisations, pinned host memory)
    # go through ONE call, which streams them rhs by rhs -- every field's upload,
    # apply and download inside the timed region, consecutive fields
    # overlapping on the two copy engines (full-duplex PCIe). Also reported:
    # one synchronous call per step (no overlap across steps).
    K = args.e2e_steps
    hin = torch.empty(NRHS * n, dtype=torch.complex128).pin_memory()
    hout = torch.empty(NRHS * n, dtype=torch.complex128).pin_memory()
    hin.copy_(U.cpu())
    hin_all = torch.empty(max(1, K) * NRHS * n, dtype=torch.complex128).pin_memory()
    hout_all = torch.empty_like(hin_all).pin_memory()
    if K > 0:
        hin_all.view(K, NRHS * n).copy_(hin.unsqueeze(0).expand(K, -1))

    def e2e_call(src, dst, nrhs):
        emie._check(L.emie_cu_apply_system_host(system.handle, ctypes.c_void_p(src.data_ptr()),
                                                ctypes.c_void_p(dst.data_ptr()), nrhs, sp))

    for _ in range(2 if K > 0 else 0):
        e2e_call(hin, hout, NRHS)
        e2e_call(hin_all, hout_all, NRHS * K)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if K > 0:
        e2e_call(hin_all, hout_all, NRHS * K)
    torch.cuda.synchronize()
    e2e_s = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
    t0 = time.perf_counter()
    for _ in range(K):
        e2e_call(hin, hout, NRHS)
    torch.cuda.synchronize()
    e2e_call_s = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
    if dist:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        dist.all_reduce(e2e_call_s, op=dist.ReduceOp.MAX)
    e2e_value = world * NRHS * K / float(e2e_s.item()) if K > 0 else None
    e2e_call_value = world * NRHS * K / float(e2e_call_s.item()) if K > 0 else None
    if K > 0:  # the streamed outputs equal the device apply's, field by field
        assert torch.equal(hout_all.view(K, NRHS * n)[-1], hout), "streamed host apply differs"
    pcie = pcie_bandwidth(hin, hout, U, W) if args.e2e_steps > 0 else None

    # the full solve the apply serves: FGMRES (restart 40, tol 1e-6) on the two
    # plane-wave right-hand sides in lockstep (cie.cpp:240-249), device resident
    solve = None
    if not args.no_solve:
        from paper_1512_06126_b200 import normal_field as NF
        rhs = np.stack([NF.build_rhs(cfg.tops, cfg.sigma, cfg.breaks, cfg.nx, cfg.ny, omega, p).reshape(-1)
                        for p in ("x", "y")])
        d_rhs = torch.from_numpy(rhs.reshape(-1)).cuda()
        # warm the stream-ordered pool for the (restart + 1)-vector bases first
        emie.fgmres_system(system, d_rhs, emie.SolverConfig(tol=1e-6, restart=40, max_iters=1))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, reps = emie.fgmres_system(system, d_rhs, emie.SolverConfig(tol=1e-6, restart=40, max_iters=2000))
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        iters = max(r.iterations for r in reps)
        # orthogonalisation traffic per iteration, 16 B x 3N per
        # vector; j averages (restart-1)/2 over full cycles. DCGS2 (default,
        # solver.cu): two tiled sweeps over the j+1 basis vectors (dots of w and
        # of v_j's delayed reorthogonalisation; v_j corrected + w projected +
        # norm) reading w in both, writing w and v_j in the second. CGS2
        # (EMIE_CU_DCGS2=0): three sweeps, w read 3x and written 2x.
        jbar = (min(40, iters) - 1) / 2.0
        dcgs2 = os.environ.get("EMIE_CU_DCGS2", "1") != "0"
        ortho_bytes = NRHS * ((2 * (jbar + 1) + 4) if dcgs2 else (3 * (jbar + 1) + 5)) * 16 * n
        solve = {"seconds": secs, "iterations": [r.iterations for r in reps],
                 "status": [r.status for r in reps], "residual": [r.residual for r in reps],
                 "tol": 1e-6, "restart": 40, "max_iters": 2000,
                 "ms_per_iteration": 1e3 * secs / max(1, iters),
                 "orthogonalisation": "DCGS2 (delayed reorthogonalisation: 2 sweeps per step)" if dcgs2
                 else "CGS2 (3 sweeps per step)",
                 "ortho_bytes_per_iteration": ortho_bytes,
                 "rhs": "x- and y-polarised plane-wave normal field (normal_field.py), both in lockstep"}
        # effective bandwidth of everything but the apply: the orthogonalisation
        # bytes over the iteration time left after the device apply step
        ortho_ms = solve["ms_per_iteration"] - ms_max / args.steps
        hbm_pk, hbm_src = peaks()
        if ortho_ms > 0:
            gbs = ortho_bytes / (ortho_ms * 1e-3) / 1e9
            solve["ortho_effective"] = {"gb_s": round(gbs, 1), "hbm_peak_gb_s": hbm_pk, "peak_source": hbm_src,
                                        "frac": round(gbs / hbm_pk, 3),
                                        "how": "ortho bytes / (solve ms per iteration - device apply ms per "
                                               "2-rhs step): the sweeps plus the small per-step kernels and gaps"}

    # roofline of the dominant kernel (the per-mode contraction)
    nz = cfg.nz
    modes = sop.qx * sop.qy
    E = sop.ex * sop.ey
    nent = 2 * nz * (2 * nz + 1)
    # blocks read per launch: every quadrant mode, or with the x <-> y symmetry
    # of a square grid (hx == hy) only the octant qmx <= qmy (operator.cu)
    octant = emie.xy_symmetric(sop)
    blocks_read = sop.qx * (sop.qx + 1) // 2 if octant else modes
    # stored entries per block: the reference's 2nz(2nz+1), or for nz 48/64 the
    # six dense nz x nz blocks the streamed contraction reads (operator.cuh)
    nent_read = 6 * nz * nz if nz in (48, 64) else nent
    bytes_ct = blocks_read * nent_read * 16 + 2 * NRHS * E * 3 * nz * 16
    flops_ct = NRHS * 72.0 * nz * nz * E
    ct_ms = ms5[2] / nprof  # per step (the passes may run once per right-hand side)
    hbm, hbm_kind = peaks()
    fp64 = ctypes.c_double(0.0)
    emie._check(L.emie_cu_probe_fp64(ctypes.byref(fp64), sp))
    # FP64 denominator: the larger of this run's probe and the nominal pipe rate
    # (SMs x 128 flop/clk x the device's maximum SM clock) -- the probe varies by a
    # few percent run to run, and a low reading must not inflate the fraction
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    fp64_probe = fp64.value
    fp64_nominal = props.multi_processor_count * 128 * props.clock_rate * 1e3 / 1e12  # clock_rate in kHz
    fp64.value = max(fp64_probe, fp64_nominal)
    achieved = bytes_ct / (ct_ms * 1e-3) / 1e9
    # template arguments as ncu names them (the last one: the sharded apply's peer epilogue, off here)
    ct_kernel = (("contract_mma_kernel<%d, %d, 0>" % (nz, int(octant))) if nz in (8, 16, 32) else
                 ("contract_rows_kernel<%d, %d, 0>" % (nz, int(octant))) if nz in (48, 64) else "contract_kernel")
    traffic = None  # dram read + write per launch, from the committed ncu --set full capture
    tpath = ROOT / "profiles" / "traffic.json"
    if tpath.exists():
        t = json.loads(tpath.read_text()).get(ct_kernel)
        if t and t.get("config") == f"cfg{args.config} nrhs={NRHS}":
            traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
    # the contraction's bound: whichever floor is longer at the measured peaks
    # (HBM bytes vs FP64 flops; 8 flops per complex multiply-add is the
    # algorithmic count, the 3-multiply form issues 6 on the DMMA pipe)
    tflops = flops_ct / (ct_ms * 1e-3) / 1e12
    hbm_view = {"achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "peak_source": hbm_kind, "bytes_per_launch": bytes_ct}
    fp64_view = {"achieved": tflops, "peak": fp64.value, "unit": "TFLOP/s",
                 "frac": tflops / fp64.value if fp64.value else None,
                 "peak_source": "max(emie_cu_probe_fp64 on this GPU: a DFMA and a DMMA m8n8k4 loop; nominal SMs x "
                                "128 flop/clk x max SM clock): MEASURED_PEAKS.json carries no FP64 figure",
                 "peak_probe": fp64_probe, "peak_nominal": fp64_nominal,
                 "flops_per_launch": flops_ct,
                 "flops": "8 per complex multiply-add of the (3nz)^2 mode matrices, all ex*ey modes",
                 "issued_dmma_frac": (0.75 * tflops / fp64.value) if (fp64.value and nz in (8, 16, 32, 48, 64)) else None,
                 "issued_dmma_frac_how": "derived: the 3-multiply complex form issues 6 of the 8 algorithmic "
                                         "flops per complex MAC (ncu sm__pipe_fp64 active is in profiles/)"}
    tensor_bound = fp64.value and flops_ct / (fp64.value * 1e12) > bytes_ct / (hbm * 1e9)
    roofline = dict(bound="tensor" if tensor_bound else "hbm", kernel=ct_kernel,
                    **(fp64_view if tensor_bound else hbm_view),
                    traffic=traffic,
                    traffic_source="profiles/traffic.json (ncu --set full, dram__bytes_read.sum + "
                                   "dram__bytes_write.sum, one launch)",
                    hbm=hbm_view, fp64=fp64_view)
    # Green's build roofline (FP64-pipe bound; the ncu-measured
    # FP64 work is authoritative): executed FP64 flops of one cfg3 build's
    # assemble stage (every launch) from the committed ncu capture over this
    # run's assemble time
    greens_roofline = None
    gpath = ROOT / "profiles" / "r02_greens_fp64.json"
    if greens_stage and gpath.exists() and args.config == 3 and fp64.value:
        gj = json.loads(gpath.read_text())
        t_as = greens_stage["assemble_kernel_ms"] * 1e-3
        p_alg = cfg.nx * cfg.ny * 451 * cfg.nz ** 2  # pair-lambda evaluations of all offsets
        ach = gj["fp64_flops_executed"] / t_as / 1e12
        greens_roofline = {
            "bound": "fp64", "kernel": gj["kernel"], "achieved": ach, "peak": fp64.value, "unit": "TFLOP/s",
            "frac": ach / fp64.value, "fp64_pipe_active_pct_ncu": gj["fp64_pipe_active_pct"],
            "flops_per_launch": gj["fp64_flops_executed"],
            "flops_how": "executed FP64 flops (2 DFMA + DADD + DMUL thread instructions, ncu) of one build's "
                         "assemble stage, all launches",
            "algorithmic": {"pair_lambda": p_alg, "flops": 140.0 * p_alg, "tflops": 140.0 * p_alg / t_as / 1e12,
                            "note": "SURVEY.md §8(d) estimate of the reference algorithm over all nx*ny offsets; "
                                    "the build computes the offsets oi <= oj (x<->y mirror) with five complex "
                                    "products per pair-lambda instead of fifteen"},
            "source": "profiles/r02_greens_fp64.json (ncu --set full)"}
    stage_names = ["fwd_x_fft", "fwd_y_fft", "contraction", "inv_y_fft", "inv_x_fft_epilogue"]
    stages = {nm: round(float(ms5[i] / nprof), 4) for i, nm in enumerate(stage_names)}  # ms per step

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            hc = host_cpu()
            d = reference_apply_rate(cfg, 4, threads=hc["threads_used"])
            times = d["times"][1:]
            cpu = {"value": NRHS * len(times) / float(np.sum(times)), "unit": UNIT,
                   "cores": d["threads"], "kind": "reference", "host": hc,
                   "sample": f"{len(times)} steps x {NRHS} applies of the reference apply(SystemOperator) "
                             f"at cfg{args.config} shape (oracle/_ref, OpenMP on the physical cores, "
                             "FFTW-API shim: no libfftw3 on the host)"}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    greens_cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            g = reference_greens_seconds(cfg, 16, threads=host_cpu()["threads_used"])
            greens_cpu = {"value_s": g["extrapolated_s"], "cores": g["threads"], "kind": "reference",
                          "sample": f"assemble_block over every {g['stride']}th offset ({g['offsets']} of "
                                    f"{g['total_offsets']}, {g['seconds']:.2f} s), extrapolated linearly"}
        except Exception as ex:  # noqa: BLE001
            greens_cpu = {"value_s": None, "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {
            "metric": metric_for(cfg), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (seeded config-3 conductivity field, seeded fields)",
            "config": config_of(args, cfg, freq if world == 1 else "one config-5 frequency per rank"),
            "operator": operator_src,
            "layout": {"operator_streamed_gb_per_step": round(blocks_read * nent_read * 16 / 1e9, 3),
                       "embedding": [sop.ex, sop.ey], "quadrant_modes": modes,
                       "contraction_blocks_read": blocks_read, "octant": octant},
            "solve": solve,
            "step_ms_percentiles": {"p10": round(float(np.percentile(per_step, 10)), 4),
                                    "p50": round(float(np.percentile(per_step, 50)), 4),
                                    "p90": round(float(np.percentile(per_step, 90)), 4)},
            "greens_build_s": greens_s,
            "library_init_s": init_s,
            "library_init": f"tiny build + apply, {LIB_POOL_RESERVE >> 30} GB reserved in the stream-ordered pool",
            "greens_build_warm_s": greens_warm_s,
            "greens_stage_ms": greens_stage,
            "greens_roofline": greens_roofline,
            "greens_cpu_baseline": greens_cpu,
            "stage_ms": stages,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_call_value, "unit": UNIT, "h2d_bytes_per_step": NRHS * n * 16,
                    "d2h_bytes_per_step": NRHS * n * 16, "pcie_gbs": pcie,
                    "how": f"one emie_cu_apply_system_host call per step ({K} steps): the step's {NRHS} "
                           "polarisation fields uploaded from pinned host memory, applied, downloaded, "
                           "all inside the timed region (FGMRES applies depend on each other, so steps "
                           "do not overlap)",
                    "streamed_independent_fields": {
                        "value": e2e_value,
                        "how": f"{K} steps x {NRHS} independent fields through one call, consecutive "
                               "fields overlapping on the copy engines (throughput for independent "
                               "sources, e.g. many right-hand sides; not a solve's dependent applies)"}},
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def pcie_bandwidth(hin, hout, din, dout):
    """Pinned-memory copy rates of this box (context for e2e, which moves
    the same bytes): H2D alone, D2H alone, both at once on two streams."""
    import torch
    nbytes = hin.numel() * hin.element_size()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, fns in (("h2d", [(s1, lambda: din.copy_(hin, non_blocking=True))]),
                      ("d2h", [(s2, lambda: hout.copy_(dout, non_blocking=True))]),
                      ("duplex", [(s1, lambda: din.copy_(hin, non_blocking=True)),
                                  (s2, lambda: hout.copy_(dout, non_blocking=True))])):
        for _ in range(2):
            for st, f in fns:
                with torch.cuda.stream(st):
                    f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            for st, f in fns:
                with torch.cuda.stream(st):
                    f()
        torch.cuda.synchronize()
        res[name] = round(3 * len(fns) * nbytes / (time.perf_counter() - t0) / 1e9, 1)
    return res


# ------------------------------------------------- strong-scaling arm ----
def run_strong(args):
    """One grid sharded over the N ranks: each rank owns a
    depth slab and a mode shard of the spectra (octant rows on square grids,
    else a quadrant-mode range); two column transposes per apply (peer stores
    or NCCL; N = 1 runs the same stages through the loopback)."""
    import torch
    import paper_1512_06126_b200 as emie
    from paper_1512_06126_b200 import configs
    from paper_1512_06126_b200 import distributed as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # EMIE_BENCH_BACKEND=gloo: a CPU-side process group (a multi-rank dry run of
    # this script on fewer GPUs; ranks share devices, their work is independent)
    backend = os.environ.get("EMIE_BENCH_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = configs.config(args.config)
    model = emie.LayeredModel(cfg.tops, cfg.sigma)
    grid = emie.make_grid(model, cfg.breaks, cfg.nx, cfg.ny, cfg.hx, cfg.hy)
    grid.sigma_a[...] = cfg.sigma_a
    # the Green's build sharded by offset (summed block arrays), each rank
    # keeping only the spectra of its quadrant-mode shard
    ex, ey = emie.smooth_embedding_size(2 * cfg.nx - 1), emie.smooth_embedding_size(2 * cfg.ny - 1)
    square = cfg.nx == cfg.ny and cfg.hx == cfg.hy and ex == ey
    if args.shard_layout == "octant" and not square:
        raise SystemExit("--shard-layout octant needs a square grid with hx == hy")
    octant = square and args.shard_layout != "quadrant"
    plan = D.ShardPlan(cfg.nx, cfg.ny, cfg.nz, ex, ey, world, octant=octant)
    torch.cuda.synchronize()
    tg0 = time.perf_counter()
    red = D.torch_block_sum() if world > 1 else D.loopback_block_sum
    (op_shard,) = D.sharded_greens_build(grid, model, cfg.omega, plan, [rank], red)
    torch.cuda.synchronize()
    greens_s = time.perf_counter() - tg0
    shard = D.cuda_shard(grid, None, plan, rank, NRHS, op_shard=op_shard)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1234)
    n = 3 * cfg.cells()
    U = rng.uniform(-1, 1, (NRHS, n)) + 1j * rng.uniform(-1, 1, (NRHS, n))
    slab = torch.from_numpy(D.slab_of(U, plan, rank, NRHS)).cuda()
    # column transposes: peer stores over NVLink into the owners' IPC-mapped
    # buffers (default) or NCCL all-to-all with pack / unpack copies
    if args.exchange == "peer":
        if world > 1:
            px = D.peer_exchange_torch(shard)
            if args.peer_sync == "host":
                px.host_barrier = dist.barrier
        else:
            (px,), _ = D.peer_loopback([shard])
        step = lambda: px.apply(slab)  # noqa: E731
    elif world > 1:
        sysd = D.DistributedSystem(shard)
        step = lambda: sysd.apply(slab)  # noqa: E731
    else:
        step = lambda: D.loopback_apply([shard], [slab])[0]  # noqa: E731
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.4)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    tmax = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
    if dist:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms = float(tmax.item())
    # end to end: the rank's slab from pinned host memory and back, each step
    hin = torch.from_numpy(D.slab_of(U, plan, rank, NRHS)).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        dev_in = hin.cuda(non_blocking=True)
        if args.exchange == "peer":
            out = px.apply(dev_in)
        else:
            out = sysd.apply(dev_in) if world > 1 else D.loopback_apply([shard], [dev_in])[0]
        hout.copy_(out)
    torch.cuda.synchronize()
    e2e_s = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
    if dist:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    check = None
    if args.exchange == "peer":
        px.check()  # a flag wait that gave up invalidates the run
    if args.check:
        out = step()
        torch.cuda.synchronize()
        parts = [None] * world
        if dist:
            dist.all_gather_object(parts, out.cpu().numpy())
        else:
            parts = [out.cpu().numpy()]
        if rank == 0:
            full_op = emie.assemble_operator(grid, model, cfg.omega)
            want = emie.apply(emie.build_system(grid, full_op), U.reshape(-1)).reshape(NRHS, -1)
            got = D.join_slabs(parts, plan, NRHS).reshape(NRHS, -1)
            check = {"max_rel_err_vs_unsharded_apply": float(np.max(np.abs(got - want)) / np.max(np.abs(want))),
                     "processes": world, "exchange": args.exchange, "peer_sync": args.peer_sync}
    if rank == 0:
        slab_bytes = hin.numel() * 16
        line = {
            "metric": metric_for(cfg), "value": NRHS * args.steps / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (seeded config conductivity field, seeded fields)",
            "config": {"workload": f"cfg{args.config} {cfg.nx}x{cfg.ny}x{cfg.nz} sharded over {world} rank(s): "
                                   "depth slabs + " + ("octant-row mode shards" if octant else "quadrant-mode shards")
                                   + ", 2 column transposes per apply "
                                   + ("as peer stores into IPC-mapped buffers (flag barriers)"
                                      if args.exchange == "peer" else "as NCCL all-to-alls"),
                       "nrhs": NRHS, "slabs": plan.z, "mode_shards": plan.q,
                       "shard_layout": "octant" if octant else "quadrant",
                       "greens_build": "sharded by offset, summed block arrays, per-rank mode-shard spectra"},
            "greens_build_s": greens_s,
            "e2e": {"value": NRHS * args.e2e_steps / float(e2e_s.item()), "unit": UNIT,
                    "h2d_bytes_per_step": slab_bytes * world, "d2h_bytes_per_step": slab_bytes * world},
            "gpu_launches": None,
            "clocks": clk,
            "check": check,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: launch the N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1; N above the visible
    device count is an error (EMIE_BENCH_BACKEND=gloo allows a dry run of the
    multi-rank path on fewer GPUs)."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if args.gpus > have and os.environ.get("EMIE_BENCH_BACKEND", "nccl") == "nccl":
        print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}), flush=True)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.strong:
        return run_strong(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
