"""Two-level nested grids on the device (SPEC.md [MODULE] nesting,
SPEC.md:363-417; paper §2.2 "usage of two (or even more) grids with different
spatial resolution", §5 global 50 m / local 12.5 m).

    coarse = CsphTvdStepper(...)                     # the global grid
    nest = NestedGrid(coarse, window=(i0, j0, ni, nj), r=4, fine_terrain=tf,
                      fine_params=pf)                # fine context + ghost band
    nest.upload(fine_state)                          # synchronized with coarse
    info = coupled_step(coarse, [nest])              # global step + subcycling + feedback

The reference has no code for this module; the operator details
(prolong_boundary, restrict_feedback, coupled_step) are documented in
csrc/swf_nest.cu and restated by the test oracle oracle/nest.py.  Each level
is a full CsphTvdStepper context, so a window runs the same fused sm_100a
step kernels as the global grid.
"""
from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi as A
from ._lib import lib
from .stepper import _ERRORS, CsphTvdStepper, raise_for
from .types import (BoundaryConfig, ConfigError, EdgeKind, FlowState, PhysicalParams, StepInfo,
                    StepperOptions, Terrain, TimestepControl)
from ._marshal import info_from_c

DEFAULT_GHOST = 2  # SPEC.md:369 "interpolation ghost band width (2 fine cells)"


def fine_shape(window: Tuple[int, int, int, int], r: int, ghost: int = DEFAULT_GHOST):
    i0, j0, ni, nj = window
    return r * ni + 2 * ghost, r * nj + 2 * ghost


def fine_origin(coarse: Terrain, window, r: int, ghost: int = DEFAULT_GHOST):
    """Physical lower-left corner of the fine grid (ghost band included)."""
    hf = coarse.h / r
    return coarse.x0 + window[0] * coarse.h - ghost * hf, coarse.y0 + window[1] * coarse.h - ghost * hf


def bathymetry_deviation(coarse: Terrain, fine: Terrain, window, r: int,
                         ghost: int = DEFAULT_GHOST) -> float:
    """Mean |restrict(b_fine) - b_coarse| over the window (SPEC.md:368,
    ingestion check; the SPEC warns above 0.5 m)."""
    i0, j0, ni, nj = window
    nxf = r * ni + 2 * ghost
    bf = fine.b.reshape(-1, nxf)[ghost:ghost + r * nj, ghost:ghost + r * ni]
    mean = bf.reshape(nj, r, ni, r).mean(axis=(1, 3))
    bc = coarse.b.reshape(coarse.ny, coarse.nx)[j0:j0 + nj, i0:i0 + ni]
    return float(np.abs(mean - bc).mean())


@dataclass
class CoupledInfo:
    tau: float
    substeps_total: int
    substeps_max: int
    fine_tau_min: float
    coarse: StepInfo
    reflux_clamp_volume: float = 0.0


class NestedGrid:
    """A fine window coupled to a global CsphTvdStepper."""

    def __init__(self, coarse: CsphTvdStepper, window: Tuple[int, int, int, int], r: int,
                 fine_terrain: Terrain, fine_params: Optional[PhysicalParams] = None,
                 control: Optional[TimestepControl] = None,
                 options: Optional[StepperOptions] = None, ghost: int = DEFAULT_GHOST,
                 two_way: bool = True, check_bathymetry: bool = True):
        self.coarse = coarse
        self.window = tuple(int(v) for v in window)
        self.r, self.ghost, self.two_way = int(r), int(ghost), bool(two_way)
        nxf, nyf = fine_shape(self.window, self.r, self.ghost)
        if fine_terrain.nx != nxf or fine_terrain.ny != nyf:
            raise ConfigError(f"nest: fine terrain must be {nxf}x{nyf} (r*window + 2*ghost)")
        if check_bathymetry:
            dev = bathymetry_deviation(coarse.terrain(), fine_terrain, self.window, self.r,
                                       self.ghost)
            if dev > 0.5:
                warnings.warn(f"nest: restricted fine bathymetry deviates from the global bed by "
                              f"{dev:.3f} m on average (> 0.5 m)")
        if options is None:  # open edges: the ghost band is overwritten every substep
            options = StepperOptions(boundaries=BoundaryConfig(EdgeKind.Open, EdgeKind.Open,
                                                               EdgeKind.Open, EdgeKind.Open))
        self.fine = CsphTvdStepper(fine_terrain, fine_params or coarse.params(),
                                   control or TimestepControl(), options)
        self._lib = lib()
        d = A.swf_nest_desc(self.window[0], self.window[1], self.window[2], self.window[3],
                            self.r, self.ghost, 1 if self.two_way else 0)
        p = C.c_void_p()
        rc = self._lib.swf_nest_create(coarse._ctx, self.fine._ctx, C.byref(d), C.byref(p))
        raise_for(rc, coarse._ctx)
        self._nest = p

    def close(self):
        if getattr(self, "_nest", None):
            self._lib.swf_nest_destroy(self._nest)
            self._nest = None
        if getattr(self, "fine", None) is not None:
            self.fine.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _rc(self, rc):
        if rc:
            msg = self._lib.swf_nest_last_error(self._nest)
            raise _ERRORS.get(rc, RuntimeError)(msg.decode() if msg else "")

    # state of the fine level
    def upload(self, state: FlowState) -> None:
        self.fine.upload(state)

    def download(self, state: FlowState) -> None:
        self.fine.download(state)

    # SPEC operations, exposed for tests and custom drivers
    def ghost_count(self) -> int:
        n = C.c_size_t()
        self._rc(self._lib.swf_nest_ghost_count(self._nest, C.byref(n)))
        return n.value

    def prolong_boundary(self, slot: int = 0) -> np.ndarray:
        """Prolong the global grid's current state into ghost slot `slot`;
        returns the (3, ghost_count) values [H, HUx, HUy]."""
        self._rc(self._lib.swf_nest_prolong(self._nest, int(slot)))
        out = np.empty(3 * self.ghost_count())
        self._rc(self._lib.swf_nest_download_ghosts(self._nest, int(slot), A.dptr(out)))
        return out.reshape(3, -1)

    def apply_ghosts(self, alpha: float) -> None:
        self._rc(self._lib.swf_nest_apply_ghosts(self._nest, float(alpha)))

    def restrict_feedback(self) -> None:
        self._rc(self._lib.swf_nest_restrict(self._nest))


def coupled_step(coarse: CsphTvdStepper, nests: Sequence[NestedGrid],
                 dt_cap: float = 0.0) -> CoupledInfo:
    """the global grid advances by tau_g; every window
    subcycles with its own CFL dt to t + tau_g (time-interpolated ghosts, the
    last substep truncated by dt_cap) and, when two-way, feeds back."""
    L = lib()
    arr = (C.c_void_p * max(1, len(nests)))(*[n._nest for n in nests])
    info = A.swf_coupled_info()
    rc = L.swf_coupled_step(coarse._ctx, arr, len(nests), float(dt_cap), C.byref(info))
    raise_for(rc, coarse._ctx)
    return CoupledInfo(info.tau, info.substeps_total, info.substeps_max, info.fine_tau_min,
                       info_from_c(info.coarse), info.reflux_clamp_volume)
