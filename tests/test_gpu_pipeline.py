"""The forward pipeline end to end on the device (SPEC.md run_forward and its
examples): a zero-contrast config reproduces the 1-D background response at
every receiver; the small anomaly config gives finite, positive apparent
resistivities with phases in range and a response that differs from the
background above the block; a rerun with a warm operator cache writes
byte-identical CSVs (determinism contract); the CLI runs the same."""
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1512_06126_b200 import pipeline as PL

pytestmark = pytest.mark.gpu
DATA = Path(__file__).resolve().parent / "data"
ROOT = Path(__file__).resolve().parent.parent


def _read(f):
    return np.loadtxt(f, delimiter=",", skiprows=1)


def test_zero_contrast_equals_background(torch_cuda, tmp_path):
    cfg = PL.load_config(DATA / "forward_small.yaml")
    cfg.blocks = []
    cfg.periods = [3.0]
    f = PL.run_forward(cfg, tmp_path / "fwd", use_cache=False, log=lambda *a: None)[0]
    g = PL.responses_1d(cfg, tmp_path / "bg")[0]
    a, b = _read(f), _read(g)
    assert np.allclose(a, b, rtol=1e-10, atol=1e-14)


def test_anomaly_run_cache_determinism_and_cli(torch_cuda, tmp_path):
    cfg = PL.load_config(DATA / "forward_small.yaml")
    cfg.cache_dir = str(tmp_path / "cache")
    f1 = PL.run_forward(cfg, tmp_path / "run1", log=lambda *a: None)
    f2 = PL.run_forward(cfg, tmp_path / "run2", log=lambda *a: None)  # operators from the cache
    assert len(list((tmp_path / "cache").iterdir())) == len(cfg.periods)
    for a, b in zip(f1, f2):
        assert a.read_bytes() == b.read_bytes()
        r = _read(a)
        rho = r[:, [11, 13]]
        phi = r[:, [12, 14]]
        assert np.all(np.isfinite(r)) and np.all(rho > 0) and np.all((phi > -180) & (phi <= 180))
        bg = _read(PL.responses_1d(cfg, tmp_path / "bg")[cfg.periods.index(r[0, 2])])
        centre = np.argmin(np.abs(r[:, 0]))
        assert abs(r[centre, 11] - bg[centre, 11]) > 1e-3 * bg[centre, 11]  # the conductive block shows
        assert abs(r[0, 11] - bg[0, 11]) < abs(r[centre, 11] - bg[centre, 11])  # and fades away from it
    cfgf = tmp_path / "c.yaml"
    shutil.copy(DATA / "forward_small.yaml", cfgf)
    out = subprocess.run([sys.executable, "-m", "paper_1512_06126_b200", "forward", str(cfgf), "--out",
                          str(tmp_path / "cli"), "--no-cache", "--log-level", "quiet"], cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    for a in f1:
        assert (tmp_path / "cli" / a.name).read_bytes() == a.read_bytes()
