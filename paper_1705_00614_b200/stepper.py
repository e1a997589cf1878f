"""CsphTvdStepper — the reference's solver API over the CUDA C ABI.

Mirrors swflood::CsphTvdStepper (/root/reference/proj/include/swflood/
stepper.hpp:76-169): same constructor arguments, set_wind / set_sources,
step(state, dt_cap), the eight stage methods, and the accessors.  Every call
goes through include/swf.h into libswflood_cuda.so; nothing is computed on
the host.

Device residency: the flow state lives on the GPU.  step() is the drop-in
form (host FlowState in, host FlowState out, one upload + one download per
call, like the reference's in-place update).  run() advances the resident
state n steps without host round trips; upload()/download() move it.
The stage methods follow the reference's call protocol: begin_step(state)
uploads `state`, the following stages work on that device copy, and
final_update(state, tau) writes the result back into `state`.
"""
from __future__ import annotations

import copy
import ctypes as C
from typing import List, Optional, Tuple

import numpy as np

from . import _abi as A
from ._lib import lib
from ._marshal import Marshalled, info_from_c
from .types import (BlockMask, ConfigError, ForceField, NumericalError, PhysicalParams,
                    SourceField, SourceSpec, StepInfo, StepperOptions, Terrain,
                    TimestepControl, WindForcing, FlowState)

_ERRORS = {A.SWF_ECONFIG: ConfigError, A.SWF_ENUMERICAL: NumericalError,
           A.SWF_ERANGE: IndexError}


def raise_for(rc: int, ctx) -> None:
    if rc == A.SWF_OK:
        return
    msg = lib().swf_last_error(ctx)
    msg = msg.decode() if msg else ""
    raise _ERRORS.get(rc, RuntimeError)(msg)


class _LiveControl:
    """control() returns a mutable reference in the reference (stepper.hpp:100)."""

    def __init__(self, owner):
        object.__setattr__(self, "_o", owner)

    def __getattr__(self, k):
        return getattr(self._o._control, k)

    def __setattr__(self, k, v):
        setattr(self._o._control, k, v)
        self._o._push_control()


class _LiveOptions:
    """options() returns a mutable reference in the reference (stepper.hpp:101)."""

    def __init__(self, owner):
        object.__setattr__(self, "_o", owner)

    def __getattr__(self, k):
        return getattr(self._o._options, k)

    def __setattr__(self, k, v):
        setattr(self._o._options, k, v)
        self._o._push_options()


class CsphTvdStepper:
    FUSED, STAGED = 0, 1

    def __init__(self, terrain: Terrain, params: PhysicalParams, control: TimestepControl,
                 options: Optional[StepperOptions] = None, *, mode: int = 0):
        options = copy.deepcopy(options) if options is not None else StepperOptions()
        self._terrain = terrain
        self._params = params
        self._control = TimestepControl(control.courant, control.dt_max, control.dt_min)
        self._options = options
        self._lib = lib()
        m = Marshalled()
        t = m.terrain(terrain)
        p = m.params(params, terrain.nx * terrain.ny)
        k = m.control(control)
        o = m.options(options)
        ctx = C.c_void_p()
        rc = self._lib.swf_create(C.byref(t), C.byref(p), C.byref(k), C.byref(o), C.byref(ctx))
        raise_for(rc, None)
        self._ctx = ctx
        self._n = terrain.nx * terrain.ny
        self._wind = WindForcing()
        self._specs: List[SourceSpec] = []
        if mode:
            self.set_mode(mode)

    # ------------------------------------------------------------------ life
    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.swf_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _rc(self, rc):
        raise_for(rc, self._ctx)

    # ---------------------------------------------------------- configuration
    def set_wind(self, wind: WindForcing) -> None:
        m = Marshalled()
        n, t, x, y = m.wind(wind)
        self._rc(self._lib.swf_set_wind(self._ctx, n, t, x, y))
        self._wind = wind

    def set_sources(self, sources: List[SourceSpec]) -> None:
        m = Marshalled()
        arr = m.sources(sources)
        self._rc(self._lib.swf_set_sources(self._ctx, len(sources), arr))
        self._specs = list(sources)

    def set_mode(self, mode: int) -> None:
        """0 = fused tile kernels (default), 1 = unfused stage kernels."""
        self._rc(self._lib.swf_set_mode(self._ctx, int(mode)))

    def set_timing(self, slots) -> None:
        """0/False: off; 1/True: timings of the last step; n > 1: per-step ring."""
        self._rc(self._lib.swf_set_timing(self._ctx, int(slots)))

    def timing_read(self, nsteps: int) -> np.ndarray:
        """(nsteps, 8) device seconds per bucket of the last nsteps fused steps."""
        out = np.zeros((nsteps, 8))
        self._rc(self._lib.swf_timing_read(self._ctx, int(nsteps), A.dptr(out)))
        return out

    def _push_control(self):
        k = Marshalled.control(self._control)
        self._rc(self._lib.swf_set_control(self._ctx, C.byref(k)))

    def _push_options(self):
        o = Marshalled.options(self._options)
        self._rc(self._lib.swf_set_options(self._ctx, C.byref(o)))

    def terrain(self) -> Terrain:
        return self._terrain

    def params(self) -> PhysicalParams:
        return self._params

    def control(self):
        return _LiveControl(self)

    def options(self):
        return _LiveOptions(self)

    # ------------------------------------------------------------- the step
    def _check_state(self, state: FlowState):
        if state.nx != self._terrain.nx or state.ny != self._terrain.ny:
            raise ConfigError("stepper: state does not match the terrain grid")
        for name in ("H", "HUx", "HUy"):
            a = getattr(state, name)
            # the native entry points read and write nx*ny doubles: a wrongly
            # sized array is a config error before any copy or native call
            if np.size(a) != self._n:
                raise ConfigError(f"stepper: state array {name} has {np.size(a)} cells, "
                                  f"the terrain grid {self._n}")
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
                    and a.size == self._n):
                setattr(state, name, np.ascontiguousarray(a, dtype=np.float64).reshape(-1).copy())

    def step(self, state: FlowState, dt_cap: float = 0.0) -> StepInfo:
        """One full step, in place on `state` (stepper.cpp:706-749)."""
        self._check_state(state)
        t = C.c_double(state.t)
        info = A.swf_step_info()
        rc = self._lib.swf_step_host(self._ctx, A.dptr(state.H), A.dptr(state.HUx),
                                     A.dptr(state.HUy), C.byref(t), float(dt_cap), C.byref(info))
        self._rc(rc)
        state.t = t.value
        return info_from_c(info)

    # resident-state API
    def upload(self, state: FlowState) -> None:
        self._check_state(state)
        self._rc(self._lib.swf_upload_state(self._ctx, A.dptr(state.H), A.dptr(state.HUx),
                                            A.dptr(state.HUy), float(state.t)))

    def download(self, state: FlowState) -> None:
        self._check_state(state)
        t = C.c_double()
        self._rc(self._lib.swf_download_state(self._ctx, A.dptr(state.H), A.dptr(state.HUx),
                                              A.dptr(state.HUy), C.byref(t)))
        state.t = t.value

    def step_resident(self, dt_cap: float = 0.0, sync: bool = True) -> Optional[StepInfo]:
        if not sync:
            self._rc(self._lib.swf_step(self._ctx, float(dt_cap), None))
            return None
        info = A.swf_step_info()
        self._rc(self._lib.swf_step(self._ctx, float(dt_cap), C.byref(info)))
        return info_from_c(info)

    def run(self, n: int, dt_cap: float = 0.0) -> Tuple[int, StepInfo]:
        """n resident steps without host synchronisation (CUDA-graph replay)."""
        done = C.c_int()
        info = A.swf_step_info()
        rc = self._lib.swf_run(self._ctx, int(n), float(dt_cap), C.byref(done), C.byref(info))
        self._rc(rc)
        return done.value, info_from_c(info)

    def last_ingest_bytes(self) -> int:
        """Host bytes the last step(state) read (see swf_last_ingest_bytes)."""
        b = C.c_longlong()
        self._rc(self._lib.swf_last_ingest_bytes(self._ctx, C.byref(b)))
        return b.value

    def last_writeback_bytes(self) -> int:
        """Host bytes the last step(state) on pinned arrays wrote back."""
        b = C.c_longlong()
        self._rc(self._lib.swf_last_writeback_bytes(self._ctx, C.byref(b)))
        return b.value

    def set_host_mirror(self, on: bool = True) -> None:
        """Opt-in host mirror (swf_set_host_mirror): step(state) on the same
        pinned arrays skips the host->device copies while the caller leaves
        them alone between steps (declare edits with host_changed())."""
        self._rc(self._lib.swf_set_host_mirror(self._ctx, 1 if on else 0))

    def host_changed(self) -> None:
        """The caller edited the mirrored arrays: the next step uploads them."""
        self._rc(self._lib.swf_host_changed(self._ctx))

    def redo_counts(self):
        """(forces, step) tiles of the last synchronised step recomputed
        exactly after a rejected speculative division."""
        a = (C.c_int * 2)()
        self._rc(self._lib.swf_debug_redo_counts(self._ctx, a))
        return a[0], a[1]

    def region_loads(self) -> str:
        """How k_step stages its tile regions: "tma" (tensor copies, even nx)
        or "threads" (per-thread loads)."""
        r = self._lib.swf_debug_region_loads(self._ctx)
        if r < 0:
            self._rc(r)
        return "tma" if r == 1 else "threads"

    def active_tiles(self):
        """(updated tiles, all tiles, cells per tile) of the last fused step."""
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        self._rc(self._lib.swf_active_tiles(self._ctx, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def sync(self) -> None:
        self._rc(self._lib.swf_sync(self._ctx))

    def stream_handle(self) -> int:
        return self._lib.swf_stream(self._ctx) or 0

    def device_state(self):
        H, X, Y = A.PD(), A.PD(), A.PD()
        self._rc(self._lib.swf_device_state(self._ctx, C.byref(H), C.byref(X), C.byref(Y)))
        return (C.cast(H, C.c_void_p).value, C.cast(X, C.c_void_p).value,
                C.cast(Y, C.c_void_p).value)

    # ------------------------------------------------------------ stage API
    def _stage(self, sid: int, arg: float = 0.0) -> float:
        tau = C.c_double(0.0)
        self._rc(self._lib.swf_stage(self._ctx, sid, float(arg), C.byref(tau)))
        return tau.value

    def begin_step(self, state: FlowState) -> None:
        self.upload(state)
        self._stage(A.STAGE_BEGIN)

    def compute_forces(self, state: FlowState) -> None:
        self._stage(A.STAGE_FORCES)

    def compute_dt(self, state: FlowState, dt_cap: float = 0.0) -> float:
        return self._stage(A.STAGE_DT, dt_cap)

    def predictor(self, state: FlowState, tau: float) -> None:
        self._stage(A.STAGE_PREDICTOR, tau)

    def mid_forces(self, state: FlowState, tau: float) -> None:
        self._stage(A.STAGE_MID_FORCES, tau)

    def corrector(self, state: FlowState, tau: float) -> None:
        self._stage(A.STAGE_CORRECTOR, tau)

    def flux(self, state: FlowState, tau: float) -> None:
        self._stage(A.STAGE_FLUX, tau)

    def final_update(self, state: FlowState, tau: float) -> None:
        self._stage(A.STAGE_FINAL, tau)
        self.download(state)

    # ----------------------------------------------------------- accessors
    def scratch(self, name: str) -> np.ndarray:
        out = np.empty(self._n, dtype=np.float64)
        self._rc(self._lib.swf_download_scratch(self._ctx, A.SCRATCH_ID[name], A.dptr(out)))
        return out

    def mask(self) -> BlockMask:
        bs = self._options.block_size
        nbx = (self._terrain.nx + bs - 1) // bs
        nby = (self._terrain.ny + bs - 1) // bs
        inn = np.zeros(nbx * nby, np.int32)
        hal = np.zeros(nbx * nby, np.int32)
        a, b = C.c_int(), C.c_int()
        self._rc(self._lib.swf_download_mask(
            self._ctx, inn.ctypes.data_as(A.PI), hal.ctypes.data_as(A.PI), C.byref(a), C.byref(b)))
        return BlockMask(bs, a.value, b.value, self._terrain.nx, self._terrain.ny, inn, hal)

    def step_sources(self) -> SourceField:
        s = self.scratch("sigma")
        return SourceField(self._terrain.nx, self._terrain.ny, s, self.scratch("src_vx"),
                           self.scratch("src_vy"), (s != 0.0).astype(np.uint8))

    def forces_n(self) -> ForceField:
        g = self.scratch
        return ForceField(self._terrain.nx, self._terrain.ny, g("fn_fx"), g("fn_fy"),
                          g("fn_fric_x"), g("fn_fric_y"), g("fn_sigma"))

    def forces_mid(self) -> ForceField:
        g = self.scratch
        return ForceField(self._terrain.nx, self._terrain.ny, g("fm_fx"), g("fm_fy"),
                          g("fm_fric_x"), g("fm_fric_y"), g("fm_sigma"))

    def half_depth(self):
        return self.scratch("half_H")

    def lagrangian_depth(self):
        return self.scratch("Ht")

    def lagrangian_momentum_x(self):
        return self.scratch("HVtx")

    def lagrangian_momentum_y(self):
        return self.scratch("HVty")

    def displacement_x(self):
        return self.scratch("drx")

    def displacement_y(self):
        return self.scratch("dry")

    def flux_mass(self):
        return self.scratch("Fh")

    def flux_momentum_x(self):
        return self.scratch("Fvx")

    def flux_momentum_y(self):
        return self.scratch("Fvy")

    def _volumes(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        self._rc(self._lib.swf_last_volumes(self._ctx, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def last_clamp_deficit(self) -> float:
        return self._volumes()[0]

    def last_source_volume(self) -> float:
        return self._volumes()[1]

    def last_boundary_outflow(self) -> float:
        return self._volumes()[2]


# ---------------------------------------------------------------------------
# free functions evaluated on the device (forcing.hpp:29-30, riemann.hpp:18-19)
# ---------------------------------------------------------------------------

def hll_face_flux_device(inputs: np.ndarray, g: float) -> np.ndarray:
    """inputs: (n,6) [hL,unL,utL,hR,unR,utR] -> (n,3) [fm,fn,ft] computed on the GPU."""
    a = np.ascontiguousarray(inputs, dtype=np.float64).reshape(-1, 6)
    out = np.empty((a.shape[0], 3))
    raise_for(lib().swf_dev_hll_face_flux(a.shape[0], A.dptr(a), float(g), A.dptr(out)), None)
    return out


def cbrt_device(x: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    out = np.empty_like(a)
    raise_for(lib().swf_dev_cbrt(a.size, A.dptr(a), A.dptr(out)), None)
    return out


def bottom_friction_device(u: np.ndarray, H: np.ndarray, g: float, n_manning: float) -> np.ndarray:
    a = np.ascontiguousarray(np.column_stack([np.asarray(u)[:, 0], np.asarray(u)[:, 1], H]),
                             dtype=np.float64)
    out = np.empty((a.shape[0], 2))
    raise_for(lib().swf_dev_bottom_friction(a.shape[0], A.dptr(a), float(g), float(n_manning),
                                            A.dptr(out)), None)
    return out
