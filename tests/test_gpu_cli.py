"""The `swflood` CLI on the GPU: validation cases (SPEC.md:513-521,
ACCEPTANCE CRITERIA 1-5), run with snapshots and summary CSV
(SPEC.md:452-466), bench (skip on/off speed-up and stage shares)."""
import csv
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
CLI = os.path.join(ROOT, "paper_1705_00614_b200", "swflood")


def run(*args, cwd=None):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=900, cwd=cwd)
    return p.returncode, p.stdout, p.stderr


def read_asc(path):
    with open(path) as f:
        hdr = {}
        for _ in range(6):
            k, v = f.readline().split()
            hdr[k.lower()] = float(v)
        data = np.loadtxt(f)
    return hdr, data[::-1].reshape(-1)  # rows north->south -> j northward


@pytest.mark.parametrize("case", ["lake-at-rest", "dam-break", "skip-equivalence", "mass-ledger",
                                  "mirror-symmetry", "zoom-mass", "speedup", "stage-shares"])
def test_validation_case_passes(case):
    rc, out, err = run("validate", case)
    assert rc == 0, out + err
    assert "PASS" in out


def test_run_writes_snapshots_and_summary(tmp_path):
    cfg = tmp_path / "lake.cfg"
    cfg.write_text("synthetic = lake 96 10\nduration = 30\ncadence = 10\n"
                   "[initial]\nmode = level\nlevel = 0.5\n")
    out = tmp_path / "out"
    rc, so, se = run("run", str(cfg), "--out", str(out))
    assert rc == 0, so + se
    rows = list(csv.DictReader(open(out / "summary.csv")))
    assert len(rows) == 4  # floor(duration / cadence) + 1
    assert float(rows[-1]["t"]) == pytest.approx(30.0, abs=1e-9)
    assert max(float(r["max_speed"]) for r in rows) <= 1e-10  # lake at rest
    hdr, H = read_asc(out / "snap00003_H.asc")
    assert hdr["ncols"] == 96 and hdr["cellsize"] == 10
    vol = H.sum() * 100.0
    assert vol == pytest.approx(float(rows[-1]["total_volume"]), rel=1e-6)  # %.6e round trip
    _, eta = read_asc(out / "snap00003_eta.asc")
    _, b = read_asc(out / "snap00000_eta.asc")
    assert np.abs(eta - b).max() <= 1e-5


def test_dry_run_eta_equals_bed(tmp_path):
    cfg = tmp_path / "dry.cfg"
    cfg.write_text("synthetic = floodplain 64 50\nduration = 5\n")
    out = tmp_path / "o"
    rc, so, se = run("run", str(cfg), "--out", str(out), "--no-skip")
    assert rc == 0, so + se
    _, eta = read_asc(out / "snap00001_eta.asc")
    _, H = read_asc(out / "snap00001_H.asc")
    assert not H.any()
    # eta = H + b = b on a dry domain, compared at %.6e
    _, eta0 = read_asc(out / "snap00000_eta.asc")
    np.testing.assert_array_equal(eta, eta0)


def test_bench_reports_speedup_and_shares(tmp_path):
    cfg = tmp_path / "b.cfg"
    cfg.write_text("synthetic = floodplain 512 50\nduration = 1\n[initial]\nmode = level\nlevel = -3\n")
    rc, out, err = run("bench", str(cfg), "--steps", "20")
    assert rc == 0, out + err
    assert "speedup from dry-block skipping" in out and "lagrange+flux+final" in out


def test_run_from_an_esri_dem(tmp_path):
    """The SPEC's run path on a real DEM file: terrain from ESRI ASCII (with a
    NODATA wall), a discharge hydrograph, snapshots."""
    n, h = 80, 10.0
    i = np.arange(n)
    b = np.add.outer(0.0 * i, 0.01 * (n - i))  # rows j, columns i: slope to the east
    b[:, 40] = -9999.0  # a NODATA wall -> impermeable high ground
    b[38:42, 40] = 0.01 * (n - 40)  # with a gap
    with open(tmp_path / "dem.asc", "w") as f:
        f.write(f"ncols {n}\nnrows {n}\nxllcorner 0\nyllcorner 0\ncellsize {h}\nNODATA_value -9999\n")
        for j in range(n - 1, -1, -1):
            f.write(" ".join(f"{v:.6f}" for v in b[j]) + "\n")
    (tmp_path / "s.cfg").write_text(
        "terrain = dem.asc\nduration = 120\ncadence = 40\n"
        "[source inflow]\nkind = discharge\ncells = 2 36 4 44\nhydrograph = 0:0, 60:50\n"
        "[boundaries]\neast = open\n")
    out = tmp_path / "o"
    rc, so, se = run("run", str(tmp_path / "s.cfg"), "--out", str(out))
    assert rc == 0, so + se
    rows = list(csv.DictReader(open(out / "summary.csv")))
    assert len(rows) == 4
    vol = [float(r["total_volume"]) for r in rows]
    assert vol[-1] > vol[0] > -1  # the inflow filled the basin
    led = float(rows[-1]["source_volume"]) - float(rows[-1]["boundary_outflow"])
    assert abs((vol[-1] - vol[0]) - (led + float(rows[-1]["clamp_deficit"]))) <= 1e-9 * max(vol[-1], 1.0)
    _, H = read_asc(out / "snap00003_H.asc")
    assert np.all(H[np.arange(n) * n + 40][:30] == 0)  # the wall stays dry below the gap
