"""Python mirror of the reference's value types and errors.

Each class restates one type of the reference's public headers
(/root/reference/proj/include/swflood/*.hpp) with the same field names,
defaults and validation messages, so code written against the reference's
C++ API reads the same here.  The arrays are numpy float64 (row-major,
k = i + j*nx, j northward, grid.hpp:15-17).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import List, Optional

import numpy as np


class ConfigError(RuntimeError):
    """errors.hpp:10-14 — bad scenario/terrain input (CLI exit code 1)."""


class NumericalError(RuntimeError):
    """errors.hpp:16-21 — tau below dt_min, CFL displacement, non-finite flux
    (CLI exit code 2)."""


@dataclass
class Vec2:
    x: float = 0.0
    y: float = 0.0


def _f64(a, n: int, what: str) -> np.ndarray:
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.size != n:
        raise ConfigError(what)
    return arr.reshape(-1)


@dataclass
class Terrain:
    """grid.hpp:18-37."""
    nx: int = 0
    ny: int = 0
    h: float = 0.0
    x0: float = 0.0
    y0: float = 0.0
    b: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def cells(self) -> int:
        return self.nx * self.ny

    def idx(self, i: int, j: int) -> int:
        return i + j * self.nx

    def contains(self, i: int, j: int) -> bool:
        return 0 <= i < self.nx and 0 <= j < self.ny

    def cell_area(self) -> float:
        return self.h * self.h

    def xc(self, i: int) -> float:
        return self.x0 + (i + 0.5) * self.h

    def yc(self, j: int) -> float:
        return self.y0 + (j + 0.5) * self.h

    def validate(self) -> None:
        """grid.cpp:13-21."""
        if self.nx < 1 or self.ny < 1:
            raise ConfigError("terrain: nx and ny must be >= 1")
        if not (self.h > 0.0):
            raise ConfigError("terrain: cell size must be positive")
        if np.asarray(self.b).size != self.cells():
            raise ConfigError("terrain: bed array size mismatch")
        bad = np.flatnonzero(~np.isfinite(np.asarray(self.b, dtype=np.float64).reshape(-1)))
        if bad.size:
            raise ConfigError(f"terrain: non-finite bed elevation at cell {int(bad[0])}")


@dataclass
class FlowState:
    """grid.hpp:42-57."""
    nx: int = 0
    ny: int = 0
    t: float = 0.0
    H: np.ndarray = field(default_factory=lambda: np.zeros(0))
    HUx: np.ndarray = field(default_factory=lambda: np.zeros(0))
    HUy: np.ndarray = field(default_factory=lambda: np.zeros(0))

    @staticmethod
    def dry(terrain: Terrain) -> "FlowState":
        n = terrain.cells()
        return FlowState(terrain.nx, terrain.ny, 0.0, np.zeros(n), np.zeros(n), np.zeros(n))

    def cells(self) -> int:
        return self.nx * self.ny

    def idx(self, i: int, j: int) -> int:
        return i + j * self.nx

    def enforce_dry_rule(self, eps_dry: float) -> None:
        """grid.cpp:33-40."""
        dry = self.H <= eps_dry
        self.HUx[dry] = 0.0
        self.HUy[dry] = 0.0

    def copy(self) -> "FlowState":
        return FlowState(self.nx, self.ny, self.t, self.H.copy(), self.HUx.copy(), self.HUy.copy())


@dataclass
class PhysicalParams:
    """grid.hpp:59-74 (defaults :60-68)."""
    g: float = 9.81
    n_manning: float = 0.02
    n_field: Optional[np.ndarray] = None
    nu: float = 0.0
    omega_z: float = 0.0
    c_a: float = 1.0e-3
    rho_air: float = 1.2
    rho_water: float = 1000.0
    eps_dry: float = 1.0e-6

    def manning(self, cell: int) -> float:
        return self.n_manning if self.n_field is None or len(self.n_field) == 0 else float(self.n_field[cell])

    def validate(self) -> None:
        """grid.cpp:42-51."""
        if not (self.g > 0.0):
            raise ConfigError("params: gravity must be positive")
        if self.n_manning < 0.0:
            raise ConfigError("params: Manning coefficient must be >= 0")
        if self.n_field is not None and np.any(np.asarray(self.n_field) < 0.0):
            raise ConfigError("params: Manning field must be >= 0")
        if self.nu < 0.0:
            raise ConfigError("params: viscosity must be >= 0")
        if not (self.rho_water > 0.0):
            raise ConfigError("params: water density must be positive")
        if self.rho_air < 0.0:
            raise ConfigError("params: air density must be >= 0")
        if not (self.eps_dry > 0.0):
            raise ConfigError("params: dry threshold must be positive")


def latitude_to_omega_z(latitude_deg: float) -> float:
    """grid.cpp:53-56."""
    return 7.2921159e-5 * math.sin(latitude_deg * math.pi / 180.0)


@dataclass
class WindSample:
    t: float = 0.0
    wx: float = 0.0
    wy: float = 0.0


@dataclass
class WindForcing:
    """grid.hpp:87-95 (time series, linear interpolation, clamped)."""
    series: List[WindSample] = field(default_factory=list)

    @staticmethod
    def constant(wx: float, wy: float) -> "WindForcing":
        return WindForcing([WindSample(0.0, wx, wy)])

    def any(self) -> bool:
        return len(self.series) > 0

    def at(self, t: float) -> Vec2:
        """grid.cpp:64-75."""
        s = self.series
        if not s:
            return Vec2()
        if len(s) == 1 or t <= s[0].t:
            return Vec2(s[0].wx, s[0].wy)
        if t >= s[-1].t:
            return Vec2(s[-1].wx, s[-1].wy)
        hi = next(k for k in range(len(s)) if t < s[k].t)
        lo = hi - 1
        a = (t - s[lo].t) / (s[hi].t - s[lo].t)
        return Vec2(s[lo].wx + a * (s[hi].wx - s[lo].wx), s[lo].wy + a * (s[hi].wy - s[lo].wy))

    def validate(self) -> None:
        """grid.cpp:77-82."""
        for k in range(1, len(self.series)):
            if not (self.series[k].t > self.series[k - 1].t):
                raise ConfigError("wind: sample times must be strictly increasing")


@dataclass
class CellRect:
    """sources.hpp:11-15 (inclusive)."""
    i0: int = 0
    j0: int = 0
    i1: int = 0
    j1: int = 0

    def count(self) -> int:
        return (self.i1 - self.i0 + 1) * (self.j1 - self.j0 + 1)


@dataclass
class HydrographSample:
    t: float = 0.0
    q: float = 0.0


class SourceKind(IntEnum):
    Discharge = 0
    Rain = 1


@dataclass
class SourceSpec:
    """sources.hpp:25-36."""
    kind: SourceKind = SourceKind.Discharge
    name: str = ""
    cells: CellRect = field(default_factory=CellRect)
    hydrograph: List[HydrographSample] = field(default_factory=list)
    rate: float = 0.0
    source_velocity: Vec2 = field(default_factory=Vec2)

    Kind = SourceKind

    def discharge_at(self, t: float) -> float:
        """sources.cpp:10-20."""
        h = self.hydrograph
        if not h:
            return 0.0
        if len(h) == 1 or t <= h[0].t:
            return h[0].q
        if t >= h[-1].t:
            return h[-1].q
        hi = next(k for k in range(len(h)) if t < h[k].t)
        lo = hi - 1
        a = (t - h[lo].t) / (h[hi].t - h[lo].t)
        return h[lo].q + a * (h[hi].q - h[lo].q)


@dataclass
class TimestepControl:
    """stepper.hpp:13-18."""
    courant: float = 0.5
    dt_max: float = 10.0
    dt_min: float = 1e-9

    def validate(self) -> None:
        """stepper.cpp:31-37."""
        if not (0.0 < self.courant < 1.0):
            raise ConfigError("timestep: Courant number must be in (0,1)")
        if not (self.dt_max > 0.0):
            raise ConfigError("timestep: dt_max must be positive")
        if not (self.dt_min > 0.0 and self.dt_min < self.dt_max):
            raise ConfigError("timestep: need 0 < dt_min < dt_max")


class EdgeKind(IntEnum):
    """stepper.hpp:20."""
    Reflective = 0
    Open = 1


@dataclass
class BoundaryConfig:
    """stepper.hpp:22-28."""
    west: EdgeKind = EdgeKind.Reflective
    east: EdgeKind = EdgeKind.Reflective
    south: EdgeKind = EdgeKind.Reflective
    north: EdgeKind = EdgeKind.Reflective

    @staticmethod
    def all(k: EdgeKind) -> "BoundaryConfig":
        return BoundaryConfig(k, k, k, k)


@dataclass
class StepperOptions:
    """stepper.hpp:59-64 (workers accepted, ignored on the GPU)."""
    block_size: int = 16
    skip_dry_blocks: bool = True
    workers: int = 1
    boundaries: BoundaryConfig = field(default_factory=BoundaryConfig)


STAGE_NAMES = ("mask", "forces", "dt", "predictor", "mid_forces", "corrector", "flux", "finalize")


@dataclass
class StageTimings:
    """stepper.hpp:31-45 (seconds)."""
    mask: float = 0.0
    forces: float = 0.0
    dt: float = 0.0
    predictor: float = 0.0
    mid_forces: float = 0.0
    corrector: float = 0.0
    flux: float = 0.0
    finalize: float = 0.0

    def total(self) -> float:
        return sum(getattr(self, k) for k in STAGE_NAMES)

    def __iadd__(self, o: "StageTimings") -> "StageTimings":
        for k in STAGE_NAMES:
            setattr(self, k, getattr(self, k) + getattr(o, k))
        return self


@dataclass
class StepInfo:
    """stepper.hpp:47-57."""
    tau: float = 0.0
    active_fraction: float = 0.0
    lagrangian_blocks: int = 0
    flux_blocks: int = 0
    total_blocks: int = 0
    timings: StageTimings = field(default_factory=StageTimings)
    clamp_deficit_volume: float = 0.0
    source_volume: float = 0.0
    boundary_outflow_volume: float = 0.0


@dataclass
class BlockMask:
    """block.hpp:20-36 (counts at block size B)."""
    block_size: int = 16
    nbx: int = 0
    nby: int = 0
    nx: int = 0
    ny: int = 0
    interior_wet: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    halo_wet: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))

    def total_blocks(self) -> int:
        return self.nbx * self.nby

    def lagrangian_active(self, ib: int) -> bool:
        return self.interior_wet[ib] > 0

    def flux_active(self, ib: int) -> bool:
        return self.interior_wet[ib] > 0 or self.halo_wet[ib] > 0

    def block_rect(self, ib: int):
        bi, bj = ib % self.nbx, ib // self.nbx
        i0, j0 = bi * self.block_size, bj * self.block_size
        return i0, j0, min(i0 + self.block_size - 1, self.nx - 1), min(j0 + self.block_size - 1, self.ny - 1)


@dataclass
class ForceField:
    """forcing.hpp:16-25."""
    nx: int = 0
    ny: int = 0
    fx: np.ndarray = None
    fy: np.ndarray = None
    fric_x: np.ndarray = None
    fric_y: np.ndarray = None
    sigma_eff: np.ndarray = None


@dataclass
class SourceField:
    """grid.hpp:99-110."""
    nx: int = 0
    ny: int = 0
    sigma: np.ndarray = None
    vx: np.ndarray = None
    vy: np.ndarray = None
    index_q: np.ndarray = None


def free_surface(state: FlowState, terrain: Terrain, i: int, j: int) -> float:
    """grid.cpp:101-106."""
    if not terrain.contains(i, j):
        raise IndexError(f"free_surface: cell ({i},{j}) outside grid")
    return float(state.H[state.idx(i, j)] + terrain.b[terrain.idx(i, j)])


def velocity(state: FlowState, params: PhysicalParams, i: int, j: int) -> Vec2:
    """grid.cpp:108-115."""
    if i < 0 or i >= state.nx or j < 0 or j >= state.ny:
        raise IndexError("velocity: cell index outside grid")
    k = state.idx(i, j)
    H = state.H[k]
    if H <= params.eps_dry:
        return Vec2()
    return Vec2(state.HUx[k] / H, state.HUy[k] / H)


def total_volume(state: FlowState, terrain: Terrain) -> float:
    """grid.cpp:117-121 (sequential sum, like the reference)."""
    s = 0.0
    for v in np.asarray(state.H, dtype=np.float64).tolist():
        s += v
    return s * terrain.cell_area()
