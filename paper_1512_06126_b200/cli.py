"""Command line of the forward pipeline (SPEC.md External Interfaces; the
reference's tools/emie_main.cpp is a placeholder):

    python -m paper_1512_06126_b200 forward <config> [--out DIR] [--no-cache]
    python -m paper_1512_06126_b200 assemble <config>      # build + cache the operators
    python -m paper_1512_06126_b200 filters <config>       # precompute the filter bank
    python -m paper_1512_06126_b200 responses1d <config> [--out DIR]
    common: --threads N (host threads of the host-side steps), --log-level {quiet,info}
"""
from __future__ import annotations

import argparse
import math
import os
import sys
from pathlib import Path

import numpy as np


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="emie-b200", description=__doc__.splitlines()[0])
    p.add_argument("command", choices=["forward", "assemble", "filters", "responses1d"])
    p.add_argument("config")
    p.add_argument("--out", default=None, help="output directory (default: next to the config)")
    p.add_argument("--no-cache", action="store_true")
    p.add_argument("--threads", type=int, default=None)
    p.add_argument("--log-level", default="info", choices=["quiet", "info"])
    a = p.parse_args(argv)
    if a.threads:
        os.environ["OMP_NUM_THREADS"] = str(a.threads)
    log = (lambda *x: None) if a.log_level == "quiet" else (lambda *x: print(*x, file=sys.stderr))
    from . import pipeline as PL
    try:
        cfg = PL.load_config(a.config)
    except (PL.ConfigError, OSError, KeyError, TypeError) as e:
        print(f"emie-b200: invalid config: {e}", file=sys.stderr)
        return 2
    out = Path(a.out) if a.out else Path(a.config).resolve().parent / "emie_out"
    try:
        if a.command == "forward":
            for f in PL.run_forward(cfg, out, use_cache=not a.no_cache, log=log):
                print(f)
        elif a.command == "responses1d":
            for f in PL.responses_1d(cfg, out):
                print(f)
        elif a.command == "assemble":
            import paper_1512_06126_b200 as emie
            if not cfg.cache_dir:
                print("emie-b200: assemble needs cache_dir in the config", file=sys.stderr)
                return 2
            model, grid = PL.build_model(cfg)
            for period in cfg.periods:
                omega = 2 * math.pi / period
                op = emie.assemble_operator(grid, model, omega, keep_blocks=True)
                f = Path(cfg.cache_dir) / f"emg1_{cfg.key(period)}.bin"
                f.parent.mkdir(parents=True, exist_ok=True)
                PL.save_operator(f, op.blocks(), cfg.nx, cfg.ny, grid.nz, omega)
                print(f)
        else:  # filters: the six weight sets of every stored offset (device design)
            import paper_1512_06126_b200 as emie
            w = np.stack([np.stack([emie.design_offset_filters(oi, oj, cfg.hx, cfg.hy)[0] for oj in range(cfg.nx)])
                          for oi in range(cfg.ny)])
            out.mkdir(parents=True, exist_ok=True)
            f = out / "filters.npz"
            np.savez_compressed(f, weights=w, hx=cfg.hx, hy=cfg.hy)
            print(f)
    except (ValueError, ArithmeticError, IndexError, RuntimeError) as e:
        print(f"emie-b200: {type(e).__name__}: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
