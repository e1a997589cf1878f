"""Synthetic scenarios of BASELINE.json's configs (seed 1705), and small
test cases.  SURVEY.md §8(d) defines them:

  C1 dam_break_1d         512x64, h=1, flat bed, H=1 left of i=256, dry or 0.1 right
  C2 circular_dam_break   2048^2, h=8, b=1e-3*x, 5 m column of radius 256 cells
  C3 floodplain           16384^2, h=50, slope + 10 seeded cosines + two meandering
                          channels, Manning field, ~35% wet, discharge ramp, drain,
                          rain, wind, Coriolis, viscosity, open east edge
  C5 floodplain           the same generator at 32768^2, h=25

Every field is a function of physical coordinates evaluated on the cells of a
`window` of the full grid, so crops (for the CPU oracle) and strips (for
multi-GPU) see exactly the values the full grid has.  Arrays are generated
with torch on the requested device (fast on the GPU for the 2^28-cell
configs) and returned as float64 numpy arrays.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from .types import (BoundaryConfig, CellRect, EdgeKind, FlowState, HydrographSample,
                    PhysicalParams, SourceKind, SourceSpec, StepperOptions, Terrain,
                    TimestepControl, Vec2, WindForcing, latitude_to_omega_z)

SEED = 1705


@dataclass
class Scenario:
    name: str
    terrain: Terrain
    params: PhysicalParams
    control: TimestepControl
    options: StepperOptions
    state: FlowState
    sources: List[SourceSpec] = field(default_factory=list)
    wind: WindForcing = field(default_factory=WindForcing)
    full_shape: Tuple[int, int] = (0, 0)
    window: Tuple[int, int, int, int] = (0, 0, 0, 0)  # i0, j0, ni, nj
    global_sources: List[SourceSpec] = field(default_factory=list)  # full-grid cells

    def cells(self) -> int:
        return self.terrain.nx * self.terrain.ny


def _torch():
    import torch
    return torch


def dam_break_1d(wet_right: bool = False, n_manning: float = 0.0, nx: int = 512,
                 ny: int = 64) -> Scenario:
    """C1: flat bed, reflective walls."""
    n = nx * ny
    b = np.zeros(n)
    H = np.zeros((ny, nx))
    H[:, : nx // 2] = 1.0
    if wet_right:
        H[:, nx // 2:] = 0.1
    st = FlowState(nx, ny, 0.0, H.reshape(-1).copy(), np.zeros(n), np.zeros(n))
    return Scenario("C1-dam-break" + ("-wet" if wet_right else "-dry"),
                    Terrain(nx, ny, 1.0, 0.0, 0.0, b), PhysicalParams(n_manning=n_manning),
                    TimestepControl(), StepperOptions(), st, full_shape=(nx, ny),
                    window=(0, 0, nx, ny))


def circular_dam_break(n: int = 2048, h: float = 8.0, radius_cells: int = 256,
                       n_manning: float = 0.03, window=None, device: str = "cpu") -> Scenario:
    """C2: sloped bed b = 1e-3 x, eta = b_center + 5 m inside the column."""
    torch = _torch()
    i0, j0, ni, nj = window if window else (0, 0, n, n)
    x = (torch.arange(i0, i0 + ni, dtype=torch.float64, device=device) + 0.5) * h
    y = (torch.arange(j0, j0 + nj, dtype=torch.float64, device=device) + 0.5) * h
    X, Y = torch.meshgrid(x, y, indexing="xy")  # (nj, ni)
    b = 1e-3 * X
    c = (n * h) / 2.0
    r = torch.sqrt((X - c) ** 2 + (Y - c) ** 2)
    eta = 1e-3 * c + 5.0
    H = torch.where(r < radius_cells * h, torch.clamp(eta - b, min=0.0), torch.zeros_like(b))
    cells = ni * nj
    st = FlowState(ni, nj, 0.0, H.reshape(-1).cpu().numpy().copy(), np.zeros(cells), np.zeros(cells))
    return Scenario("C2-circular-dam-break", Terrain(ni, nj, h, i0 * h, j0 * h,
                                                     b.reshape(-1).cpu().numpy().copy()),
                    PhysicalParams(n_manning=n_manning), TimestepControl(), StepperOptions(), st,
                    full_shape=(n, n), window=(i0, j0, ni, nj))


def _cosines(seed: int, L: float):
    rng = np.random.default_rng(seed)
    terms = []
    for _ in range(10):
        lam = L * rng.uniform(1.0 / 16.0, 1.0 / 3.0)
        ang = rng.uniform(0.0, math.pi)
        k = 2.0 * math.pi / lam
        terms.append((k * math.cos(ang), k * math.sin(ang), rng.uniform(0.0, 2.0 * math.pi)))
    return terms


def _floodplain_fields(X, Y, L: float, h: float, seed: int):
    """Bed, channel mask and Manning field at physical coordinates X, Y."""
    torch = _torch()
    b = 5e-5 * (L - X)  # slope 5e-5, descending eastward
    noise = torch.zeros_like(X)
    for kx, ky, ph in _cosines(seed, L):
        noise += 0.5 * torch.cos(kx * X + ky * Y + ph)  # 10 x 0.5 m = 5 m amplitude
    b = b + noise
    # main channel: 25 m deep, ~20 cells wide, meandering west -> east
    yc = 0.5 * L + (L / 6.0) * torch.sin(2.0 * math.pi * X / (L / 3.0))
    w1 = 10.0 * h
    p1 = torch.clamp(1.0 - ((Y - yc) / w1) ** 2, min=0.0)
    # secondary channel: 8 m deep, ~6 cells wide
    yc2 = 0.25 * L + (L / 10.0) * torch.sin(2.0 * math.pi * X / (L / 5.0) + 1.0)
    w2 = 3.0 * h
    p2 = torch.clamp(1.0 - ((Y - yc2) / w2) ** 2, min=0.0)
    b = b - 25.0 * p1 - 8.0 * p2
    chan = (p1 > 0) | (p2 > 0)
    nfield = torch.where(chan, torch.full_like(X, 0.025), torch.full_like(X, 0.04))
    return b, noise, chan, nfield


def _flood_offset(L: float, h: float, seed: int, wet_fraction: float = 0.35) -> float:
    """Water-plane offset giving ~35% wet cells, from a fixed coarse sample of
    the full-domain generator (so every crop uses the same plane)."""
    torch = _torch()
    m = 512
    s = (torch.arange(m, dtype=torch.float64) + 0.5) * (L / m)
    X, Y = torch.meshgrid(s, s, indexing="xy")
    b, noise, chan, _ = _floodplain_fields(X, Y, L, h, seed)
    rel = (b - 5e-5 * (L - X)).reshape(-1)
    return float(torch.quantile(rel, wet_fraction))


def floodplain(n: int = 16384, h: float = 50.0, window=None, device: str = "cpu",
               seed: int = SEED) -> Scenario:
    """C3 (n=16384, h=50) and C5 (n=32768, h=25): Volga-Akhtuba-like floodplain."""
    torch = _torch()
    L = n * h
    i0, j0, ni, nj = window if window else (0, 0, n, n)
    x = (torch.arange(i0, i0 + ni, dtype=torch.float64, device=device) + 0.5) * h
    y = (torch.arange(j0, j0 + nj, dtype=torch.float64, device=device) + 0.5) * h
    X, Y = torch.meshgrid(x, y, indexing="xy")
    b, noise, chan, nfield = _floodplain_fields(X, Y, L, h, seed)
    off = _flood_offset(L, h, seed)
    eta0 = 5e-5 * (L - X) + off
    H = torch.clamp(eta0 - b, min=0.0)
    H = torch.where(H > 1e-6, H, torch.zeros_like(H))
    cells = ni * nj
    to_np = lambda t: t.reshape(-1).cpu().numpy().copy()
    terrain = Terrain(ni, nj, h, i0 * h, j0 * h, to_np(b))
    params = PhysicalParams(n_manning=0.04, n_field=to_np(nfield), nu=1.0,
                            omega_z=latitude_to_omega_z(48.7))
    opts = StepperOptions(boundaries=BoundaryConfig(EdgeKind.Reflective, EdgeKind.Open,
                                                    EdgeKind.Reflective, EdgeKind.Reflective))
    st = FlowState(ni, nj, 0.0, to_np(H), np.zeros(cells), np.zeros(cells))
    # sources in FULL-grid cells, clipped to the window
    jc = int((0.5 * L) / h)
    jd = int((0.5 * L + (L / 6.0) * math.sin(2.0 * math.pi * (L - 3 * h) / (L / 3.0))) / h)
    full_specs = [
        SourceSpec(SourceKind.Discharge, "upstream", CellRect(1, jc - 5, 4, jc + 5),
                   [HydrographSample(0.0, 0.0), HydrographSample(3600.0, 1.0e5)], 0.0,
                   Vec2(1.0, 0.0)),
        SourceSpec(SourceKind.Discharge, "drain", CellRect(n - 5, jd - 5, n - 2, jd + 5),
                   [HydrographSample(0.0, -3.0e4)], 0.0, Vec2(0.0, 0.0)),
        SourceSpec(SourceKind.Rain, "rain", CellRect(n // 8, (5 * n) // 8, n // 4, (3 * n) // 4),
                   [], 1.0e-6, Vec2(0.0, 0.0)),
    ]
    specs = []
    for s in full_specs:
        a0, b0 = max(s.cells.i0, i0), max(s.cells.j0, j0)
        a1, b1 = min(s.cells.i1, i0 + ni - 1), min(s.cells.j1, j0 + nj - 1)
        if a0 <= a1 and b0 <= b1:
            specs.append(SourceSpec(s.kind, s.name, CellRect(a0 - i0, b0 - j0, a1 - i0, b1 - j0),
                                    list(s.hydrograph), s.rate, s.source_velocity))
    name = "C3-floodplain" if n == 16384 else ("C5-floodplain" if n == 32768 else f"floodplain-{n}")
    return Scenario(name, terrain, params, TimestepControl(), opts, st, specs,
                    WindForcing.constant(5.0, 2.0), full_shape=(n, n), window=(i0, j0, ni, nj),
                    global_sources=full_specs)


@dataclass
class NestedScenario:
    """C4: a global scenario plus one fine window."""
    coarse: Scenario
    fine: Scenario
    window: Tuple[int, int, int, int]  # coarse cells i0, j0, ni, nj
    r: int
    ghost: int


def nested_floodplain(n: int = 4096, h: float = 50.0, window=(1536, 1536, 1024, 1024),
                      r: int = 4, ghost: int = 2, device: str = "cpu",
                      seed: int = SEED) -> NestedScenario:
    """C4 (BASELINE.json configs[3]): the floodplain
    generator on a coarse n x n grid at h, and the SAME generator (same
    physical features, feature scale h) sampled on the fine window at h/r plus
    the ghost band.  Sources are clipped to the window and rescaled to fine
    cells (sigma = q / (count h_f^2) is unchanged); wind, Coriolis, viscosity
    and the Manning field are shared."""
    torch = _torch()
    coarse = floodplain(n, h, device=device, seed=seed)
    coarse.name = f"C4-nested-coarse-{n}"
    i0, j0, ni, nj = window
    L = n * h
    hf = h / r
    nxf, nyf = r * ni + 2 * ghost, r * nj + 2 * ghost
    x0f = i0 * h - ghost * hf
    y0f = j0 * h - ghost * hf
    x = x0f + (torch.arange(nxf, dtype=torch.float64, device=device) + 0.5) * hf
    y = y0f + (torch.arange(nyf, dtype=torch.float64, device=device) + 0.5) * hf
    X, Y = torch.meshgrid(x, y, indexing="xy")
    b, noise, chan, nfield = _floodplain_fields(X, Y, L, h, seed)
    off = _flood_offset(L, h, seed)
    H = torch.clamp(5e-5 * (L - X) + off - b, min=0.0)
    H = torch.where(H > 1e-6, H, torch.zeros_like(H))
    to_np = lambda t: t.reshape(-1).cpu().numpy().copy()
    cells = nxf * nyf
    terrain = Terrain(nxf, nyf, hf, x0f, y0f, to_np(b))
    params = PhysicalParams(n_manning=0.04, n_field=to_np(nfield), nu=coarse.params.nu,
                            omega_z=coarse.params.omega_z)
    opts = StepperOptions(boundaries=BoundaryConfig(EdgeKind.Open, EdgeKind.Open, EdgeKind.Open,
                                                    EdgeKind.Open))
    st = FlowState(nxf, nyf, 0.0, to_np(H), np.zeros(cells), np.zeros(cells))
    # ingestion consistency: the global bed over the window is
    # the block mean of the fine bed (summed in restrict_feedback's order), so
    # restricting a lake at rest gives the coarse lake at rest
    bf = terrain.b.reshape(nyf, nxf)[ghost:ghost + r * nj, ghost:ghost + r * ni]
    blk = bf.reshape(nj, r, ni, r)
    acc = np.zeros((nj, ni))
    for bb in range(r):
        for aa in range(r):
            acc = acc + blk[:, bb, :, aa]
    Bc = coarse.terrain.b.reshape(n, n)
    Bc[j0:j0 + nj, i0:i0 + ni] = acc / float(r * r)
    xc = (np.arange(i0, i0 + ni) + 0.5) * h
    eta_c = 5e-5 * (L - xc)[None, :] + off
    Hc = np.maximum(eta_c - Bc[j0:j0 + nj, i0:i0 + ni], 0.0)
    coarse.state.H.reshape(n, n)[j0:j0 + nj, i0:i0 + ni] = np.where(Hc > 1e-6, Hc, 0.0)
    specs = []
    for sp in coarse.global_sources:
        a0, b0 = max(sp.cells.i0, i0), max(sp.cells.j0, j0)
        a1, b1 = min(sp.cells.i1, i0 + ni - 1), min(sp.cells.j1, j0 + nj - 1)
        if a0 <= a1 and b0 <= b1:
            rect = CellRect(ghost + (a0 - i0) * r, ghost + (b0 - j0) * r,
                            ghost + (a1 - i0 + 1) * r - 1, ghost + (b1 - j0 + 1) * r - 1)
            specs.append(SourceSpec(sp.kind, sp.name, rect, list(sp.hydrograph), sp.rate,
                                    sp.source_velocity))
    fine = Scenario(f"C4-nested-fine-r{r}", terrain, params, TimestepControl(), opts, st, specs,
                    coarse.wind, full_shape=(nxf, nyf), window=(0, 0, nxf, nyf))
    return NestedScenario(coarse, fine, tuple(window), r, ghost)


def lake_at_rest(n: int = 128, h: float = 10.0, level: float = 0.0, seed: int = SEED) -> Scenario:
    """SPEC.md:540 acceptance 1: still lake over a seeded bumpy bed."""
    torch = _torch()
    L = n * h
    s = (torch.arange(n, dtype=torch.float64) + 0.5) * h
    X, Y = torch.meshgrid(s, s, indexing="xy")
    b = torch.zeros_like(X)
    for kx, ky, ph in _cosines(seed, L):
        b += 0.5 * torch.cos(kx * X + ky * Y + ph)
    H = torch.clamp(level - b, min=0.0)
    cells = n * n
    st = FlowState(n, n, 0.0, H.reshape(-1).numpy().copy(), np.zeros(cells), np.zeros(cells))
    return Scenario("lake-at-rest", Terrain(n, n, h, 0.0, 0.0, b.reshape(-1).numpy().copy()),
                    PhysicalParams(), TimestepControl(), StepperOptions(), st,
                    full_shape=(n, n), window=(0, 0, n, n))


def window_of(sc: Scenario, w0: int, w1: int) -> Scenario:
    """Rows [w0, w1) of a full-grid scenario (a strip's local window: terrain,
    Manning field, state); the sources stay in full-grid cells
    (global_sources), as strips take them, and the wind is shared."""
    import copy
    T = sc.terrain
    nx = T.nx
    sl = slice(w0 * nx, w1 * nx)
    p = copy.deepcopy(sc.params)
    if p.n_field is not None and len(p.n_field):
        p.n_field = np.array(p.n_field[sl], copy=True)
    st = sc.state
    ws = FlowState(nx, w1 - w0, st.t, np.array(st.H[sl]), np.array(st.HUx[sl]),
                   np.array(st.HUy[sl]))
    return Scenario(sc.name, Terrain(nx, w1 - w0, T.h, T.x0, T.y0 + w0 * T.h,
                                     np.array(T.b[sl])), p, sc.control, sc.options, ws,
                    wind=sc.wind, full_shape=(nx, T.ny), window=(0, w0, nx, w1 - w0),
                    global_sources=list(sc.global_sources or sc.sources))


def build(config: str, device: str = "cpu", window=None) -> Scenario:
    """Scenario for a BASELINE.json config id: C1, C1w, C2, C3, C5."""
    if config in ("C1", "C1-dry"):
        return dam_break_1d(False, 0.0)
    if config in ("C1w", "C1-wet"):
        return dam_break_1d(True, 0.02)
    if config == "C2":
        return circular_dam_break(window=window, device=device)
    if config == "C3":
        return floodplain(16384, 50.0, window=window, device=device)
    if config == "C4":
        return nested_floodplain(device=device)
    if config == "C5":
        return floodplain(32768, 25.0, window=window, device=device)
    if config == "C5W":  # weak scaling, one GPU's share: 32768 x 4096 rows of C5
        return floodplain(32768, 25.0, window=window or (0, 0, 32768, WEAK_ROWS), device=device)
    raise ValueError(config)


# rows per GPU of the weak-scaling configuration (BASELINE.json config 5)
WEAK_ROWS = 4096


def clip_sources(specs, nx: int, ny: int):
    """Global source specs restricted to an nx x ny domain (the weak-scaling
    grids are the first rows of the C5 generator; sources outside are dropped,
    partial ones clipped)."""
    out = []
    for s in specs:
        a0, b0 = max(s.cells.i0, 0), max(s.cells.j0, 0)
        a1, b1 = min(s.cells.i1, nx - 1), min(s.cells.j1, ny - 1)
        if a0 <= a1 and b0 <= b1:
            out.append(SourceSpec(s.kind, s.name, CellRect(a0, b0, a1, b1), list(s.hydrograph),
                                  s.rate, s.source_velocity))
    return out
