"""Seeded random small scenarios for parity fuzzing (test infrastructure).

Every knob the step path has is drawn at random: grid shape (odd and even,
partial tiles), cell size, bed (slope + cosines + noise), wet fraction,
films near eps_dry, momenta, Manning constant or field (or none), viscosity,
Coriolis, a wind series, 0-3 sources (discharge with positive or negative
hydrographs, rain; overlapping, clipped to the grid), Courant number, dt_max,
block size (dividing and not dividing the 32x16 tile), dry-block skipping,
and each edge reflective or open.
"""
import math

import numpy as np

from paper_1705_00614_b200.scenarios import Scenario
from paper_1705_00614_b200.types import (BoundaryConfig, CellRect, EdgeKind, FlowState,
                                         HydrographSample, PhysicalParams, SourceKind,
                                         SourceSpec, StepperOptions, Terrain, TimestepControl,
                                         Vec2, WindForcing, WindSample, latitude_to_omega_z)


def random_scenario(seed: int) -> Scenario:
    rng = np.random.default_rng(10_000 + seed)
    nx = int(rng.integers(6, 150))
    ny = int(rng.integers(6, 150))
    h = float(rng.choice([0.5, 2.0, 7.5, 25.0, 50.0]))
    x = (np.arange(nx) + 0.5) * h
    y = (np.arange(ny) + 0.5) * h
    X, Y = np.meshgrid(x, y, indexing="xy")
    L = max(nx, ny) * h
    b = rng.uniform(-2e-3, 2e-3) * X + rng.uniform(-2e-3, 2e-3) * Y
    for _ in range(int(rng.integers(1, 5))):
        kx, ky = rng.uniform(0.5, 6.0, 2) * 2 * math.pi / L
        b += rng.uniform(0.05, 2.0) * np.cos(kx * X + ky * Y + rng.uniform(0, 2 * math.pi))
    b += rng.normal(0, 0.01, b.shape) * rng.integers(0, 2)
    level = float(np.quantile(b, rng.uniform(0.05, 0.95)))
    H = np.maximum(level - b, 0.0)
    # films around eps_dry and a few isolated wet / dry cells
    eps = 1e-6
    m = rng.random(H.shape)
    H[m < 0.02] = eps * rng.choice([0.5, 1.0, 2.0])
    H[(m > 0.98)] = 0.0
    vmax = float(rng.choice([0.0, 0.3, 1.5]))
    U = vmax * np.cos(2 * math.pi * X / L + rng.uniform(0, 6)) * (rng.random(H.shape) * 0.5 + 0.75)
    V = vmax * np.sin(2 * math.pi * Y / L + rng.uniform(0, 6)) * (rng.random(H.shape) * 0.5 + 0.75)
    HUx = np.where(H > eps, H * U, 0.0)
    HUy = np.where(H > eps, H * V, 0.0)
    n_cells = nx * ny

    p = PhysicalParams()
    mode = int(rng.integers(0, 3))
    if mode == 0:
        p.n_manning = 0.0
    elif mode == 1:
        p.n_manning = float(rng.uniform(0.01, 0.06))
    else:
        p.n_field = rng.uniform(0.0, 0.06, n_cells)
    p.nu = float(rng.choice([0.0, rng.uniform(0.1, 3.0)]))
    p.omega_z = latitude_to_omega_z(float(rng.uniform(-70, 70))) if rng.random() < 0.5 else 0.0

    ctl = TimestepControl(courant=float(rng.uniform(0.2, 0.9)),
                          dt_max=float(rng.choice([10.0, 1.0, 0.05])), dt_min=1e-9)
    opt = StepperOptions()
    opt.block_size = int(rng.choice([1, 2, 4, 7, 8, 16, 32]))
    opt.skip_dry_blocks = bool(rng.random() < 0.7)
    edge = lambda: EdgeKind.Open if rng.random() < 0.4 else EdgeKind.Reflective
    opt.boundaries = BoundaryConfig(edge(), edge(), edge(), edge())

    wind = WindForcing()
    if rng.random() < 0.5:
        ts = np.sort(rng.uniform(0, 30, int(rng.integers(1, 4))))
        wind = WindForcing([WindSample(float(t), float(rng.uniform(-15, 15)),
                                       float(rng.uniform(-15, 15))) for t in ts])

    sources = []
    for s in range(int(rng.integers(0, 4))):
        i0 = int(rng.integers(0, nx))
        j0 = int(rng.integers(0, ny))
        i1 = min(nx - 1, i0 + int(rng.integers(0, 8)))
        j1 = min(ny - 1, j0 + int(rng.integers(0, 8)))
        spec = SourceSpec(name=f"s{s}", cells=CellRect(i0, j0, i1, j1),
                          source_velocity=Vec2(float(rng.uniform(-1, 1)), float(rng.uniform(-1, 1))))
        if rng.random() < 0.6:
            spec.kind = SourceKind.Discharge
            ts = np.sort(rng.uniform(0, 20, int(rng.integers(1, 4))))
            sign = -1.0 if rng.random() < 0.3 else 1.0
            spec.hydrograph = [HydrographSample(float(t), sign * float(rng.uniform(0, 5 * h * h)))
                               for t in ts]
        else:
            spec.kind = SourceKind.Rain
            spec.rate = float(rng.uniform(0, 1e-3))
        sources.append(spec)

    st = FlowState(nx, ny, 0.0, H.reshape(-1).copy(), HUx.reshape(-1).copy(), HUy.reshape(-1).copy())
    return Scenario(f"fuzz{seed}", Terrain(nx, ny, h, 0.0, 0.0, b.reshape(-1).copy()), p, ctl,
                    opt, st, sources=sources, wind=wind, full_shape=(nx, ny),
                    window=(0, 0, nx, ny))


INFO_FIELDS = ("tau", "active_fraction", "lagrangian_blocks", "flux_blocks", "total_blocks",
               "clamp_deficit_volume", "source_volume", "boundary_outflow_volume")


def _same(x, y):
    return np.float64(x).tobytes() == np.float64(y).tobytes()


def run_pair(a, b, sa, sb, steps, dt_cap=0.0):
    """Step two steppers side by side: every StepInfo field (timings aside)
    bitwise equal, and an abort at the same step with the same type and
    message.  Returns (steps done, abort message or None)."""
    for k in range(steps):
        ea = eb = ia = ib = None
        try:
            ia = a.step(sa, dt_cap)
        except Exception as e:  # noqa: BLE001 -- compared below
            ea = e
        try:
            ib = b.step(sb, dt_cap)
        except Exception as e:  # noqa: BLE001
            eb = e
        if ea is not None or eb is not None:
            assert type(ea).__name__ == type(eb).__name__, (k, ea, eb)
            assert str(ea) == str(eb), (k, str(ea), str(eb))
            return k, str(ea)
        for f in INFO_FIELDS:
            assert _same(getattr(ia, f), getattr(ib, f)), (k, f, getattr(ia, f), getattr(ib, f))
    return steps, None



def window(sc: Scenario, w0: int, w1: int) -> Scenario:
    """Rows [w0, w1) of a full-grid scenario (scenarios.window_of)."""
    from paper_1705_00614_b200.scenarios import window_of
    return window_of(sc, w0, w1)
