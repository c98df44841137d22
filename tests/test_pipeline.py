"""Forward pipeline host logic: config parsing and
validation, block painting, the EMG1 snapshot format (read back by the
reference's own load_operator through oracle/_ref), MT responses and the CSV
contract. GPU runs of the whole pipeline are in test_gpu_pipeline.py."""
import math
from pathlib import Path

import numpy as np
import pytest

from paper_1512_06126_b200 import normal_field as NF
from paper_1512_06126_b200 import pipeline as PL

DATA = Path(__file__).resolve().parent / "data"


def test_parse_config_and_blocks():
    cfg = PL.load_config(DATA / "forward_small.yaml")
    assert cfg.tops == [0.0, 1000.0, 11000.0] and cfg.sigma[0] == 0 and cfg.sigma[1] == 0.01
    assert (cfg.nx, cfg.ny, len(cfg.breaks) - 1) == (8, 8, 4)
    assert cfg.receivers.shape == (7, 3) and np.all(cfg.receivers[:, 2] == 0)
    model, grid = PL.build_model(cfg)
    sa = np.asarray(grid.sigma_a)
    assert np.all(sa[:3, 2:6, 2:6] == 1.0)           # inside the block (z 100-400, x,y -500..500)
    assert np.all(sa[3] == 0.01) and sa[0, 0, 0] == 0.01
    bad = dict(layers=[{"top_depth_m": 0.0, "conductivity_S_per_m": 0.01}], grid={"nx": 2, "ny": 2, "hx_m": 1,
               "hy_m": 1, "z_breaks_m": [0, 1], "nz": 3}, periods_s=[1.0])
    with pytest.raises(PL.ConfigError):
        PL.parse_config(bad)
    with pytest.raises(PL.ConfigError):
        PL.parse_config({"grid": {}})


def test_mt_responses_halfspace_and_csv():
    sigma, period = 0.02, 10.0
    omega = 2 * math.pi / period
    recs = np.array([[0.0, 0.0, 0.0], [100.0, -50.0, 0.0]])
    E, H = NF.normal_fields([0.0], [0.0, sigma], omega, recs)
    res = PL.mt_responses(E, H, recs, omega)
    for r in res:
        assert abs(r.rho_xy * sigma - 1) < 1e-3 and abs(r.rho_yx * sigma - 1) < 1e-3
        assert abs(r.phi_xy - 45.0) < 0.05 and abs(abs(r.phi_yx) - 135.0) < 0.05 or abs(r.phi_yx - 45.0) < 0.05
        assert abs(r.Z[0, 0]) < 1e-12 * abs(r.Z[0, 1])
    text = PL.csv_rows(res)
    lines = text.strip().split("\n")
    assert lines[0] == PL.CSV_HEADER and len(lines) == 3
    assert all(len(l.split(",")) == 15 for l in lines[1:])
    assert all("e" in v and len(v.split("e")[0].replace("-", "").replace(".", "")) == 9 for v in lines[1].split(","))
    with pytest.raises(ArithmeticError):
        PL.mt_responses(E, np.zeros_like(H), recs, omega)


def test_emg1_roundtrip_and_reference_reader(tmp_path):
    rng = np.random.default_rng(2)
    nx, ny, nz = 3, 2, 2
    blocks = rng.standard_normal((ny, nx, 2 * nz * (2 * nz + 1))) + 1j * rng.standard_normal((ny, nx, 20))
    f = tmp_path / "op.bin"
    PL.save_operator(f, blocks, nx, ny, nz, 0.5)
    b2, om = PL.load_operator(f, nx, ny, nz)
    assert om == 0.5 and np.array_equal(b2, blocks)
    assert PL.load_operator(tmp_path / "absent.bin", nx, ny, nz) is None
    (tmp_path / "trunc.bin").write_bytes(f.read_bytes()[:100])
    assert PL.load_operator(tmp_path / "trunc.bin", nx, ny, nz) is None
    import json
    import ref_binding as R
    if R.TOOL.exists():  # the reference's own load_operator reads the file and re-saves the same bytes
        resaved = tmp_path / "resaved.bin"
        d = json.loads(R.run_tool("snapshot-check", f, resaved))
        assert d["loaded"] and (d["nx"], d["ny"], d["nz"]) == (nx, ny, nz) and d["omega"] == 0.5
        assert resaved.read_bytes() == f.read_bytes()
