"""Python value types -> C ABI structs (include/swf.h), keeping buffers alive."""
import ctypes as C

import numpy as np

from . import _abi as A
from .types import (ConfigError, EdgeKind, PhysicalParams, SourceKind, SourceSpec,
                    StepInfo, StepperOptions, StageTimings, Terrain, TimestepControl,
                    WindForcing, STAGE_NAMES)


class Marshalled:
    """Holds ctypes structs plus the numpy arrays they point into."""

    def __init__(self):
        self.keep = []

    def arr(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        self.keep.append(a)
        return a

    def terrain(self, t: Terrain) -> A.swf_terrain:
        b = self.arr(t.b)
        if b.size != t.nx * t.ny:
            raise ConfigError("terrain: bed array size mismatch")
        return A.swf_terrain(int(t.nx), int(t.ny), float(t.h), float(t.x0), float(t.y0), A.dptr(b))

    def params(self, p: PhysicalParams, ncells: int) -> A.swf_params:
        nf = A.PD()
        if p.n_field is not None and len(p.n_field) > 0:
            a = self.arr(p.n_field)
            if a.size != ncells:
                raise ConfigError("stepper: Manning field size mismatch")
            nf = A.dptr(a)
        return A.swf_params(p.g, p.n_manning, p.nu, p.omega_z, p.c_a, p.rho_air,
                            p.rho_water, p.eps_dry, nf)

    @staticmethod
    def control(k: TimestepControl) -> A.swf_control:
        return A.swf_control(k.courant, k.dt_max, k.dt_min)

    @staticmethod
    def options(o: StepperOptions) -> A.swf_options:
        b = o.boundaries
        return A.swf_options(int(o.block_size), int(bool(o.skip_dry_blocks)), int(o.workers),
                             int(b.west), int(b.east), int(b.south), int(b.north))

    def sources(self, specs):
        arr = (A.swf_source * max(1, len(specs)))()
        for k, s in enumerate(specs):
            ht = self.arr([h.t for h in s.hydrograph]) if s.hydrograph else None
            hq = self.arr([h.q for h in s.hydrograph]) if s.hydrograph else None
            arr[k] = A.swf_source(int(s.kind), s.cells.i0, s.cells.j0, s.cells.i1, s.cells.j1,
                                  len(s.hydrograph), A.dptr(ht), A.dptr(hq), float(s.rate),
                                  float(s.source_velocity.x), float(s.source_velocity.y))
        self.keep.append(arr)
        return arr

    def wind(self, w: WindForcing):
        t = self.arr([s.t for s in w.series]) if w.series else None
        x = self.arr([s.wx for s in w.series]) if w.series else None
        y = self.arr([s.wy for s in w.series]) if w.series else None
        return len(w.series), A.dptr(t), A.dptr(x), A.dptr(y)


def info_from_c(ci: A.swf_step_info) -> StepInfo:
    tm = StageTimings(*[ci.timings[k] for k in range(8)])
    return StepInfo(ci.tau, ci.active_fraction, ci.lagrangian_blocks, ci.flux_blocks,
                    ci.total_blocks, tm, ci.clamp_deficit_volume, ci.source_volume,
                    ci.boundary_outflow_volume)
