"""TEST INFRASTRUCTURE ONLY.  ctypes driver for the checker ABI
(oracle/swf_oracle.h) of either
  * liborc.so            — the plain-C restatement (oracle/swf_oracle.c), or
  * _ref/libswflood_ref.so — the real reference compiled from /root/reference.

OracleStepper exposes the same methods as the product's CsphTvdStepper
(paper_1705_00614_b200/stepper.py), so parity tests run one scenario through
both and compare arrays bit for bit.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1705_00614_b200 import _abi as A
from paper_1705_00614_b200._marshal import Marshalled, info_from_c
from paper_1705_00614_b200.types import (BlockMask, ConfigError, FlowState, ForceField,
                                         NumericalError, SourceField, StepperOptions)

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libswflood_ref.so")
REFERENCE_SRC = "/root/reference/proj"

_libs = {}


def build(ref: bool = True) -> None:
    """Compile the C restatement and, when /root/reference exists, the real
    reference (oracle/Makefile)."""
    targets = ["orc"]
    if ref and os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _declare(lib):
    P, I, D = C.c_void_p, C.c_int, C.c_double
    PD, PI = A.PD, A.PI
    sig = {
        "orc_create": (I, [C.POINTER(A.swf_terrain), C.POINTER(A.swf_params),
                           C.POINTER(A.swf_control), C.POINTER(A.swf_options), C.POINTER(P)]),
        "orc_destroy": (None, [P]),
        "orc_last_error": (C.c_char_p, [P]),
        "orc_set_wind": (I, [P, I, PD, PD, PD]),
        "orc_set_sources": (I, [P, I, C.POINTER(A.swf_source)]),
        "orc_set_control": (I, [P, C.POINTER(A.swf_control)]),
        "orc_set_options": (I, [P, C.POINTER(A.swf_options)]),
        "orc_set_state": (I, [P, PD, PD, PD, D]),
        "orc_get_state": (I, [P, PD, PD, PD, PD]),
        "orc_step": (I, [P, D, C.POINTER(A.swf_step_info)]),
        "orc_run": (I, [P, I, D, PI, C.POINTER(A.swf_step_info)]),
        "orc_stage": (I, [P, I, D, PD]),
        "orc_scratch": (I, [P, I, PD]),
        "orc_mask": (I, [P, PI, PI, PI, PI]),
        "orc_face_fm": (I, [P, I, PD]),
        "orc_volumes": (I, [P, PD, PD, PD]),
        "orc_cbrt": (D, [D]),
        "orc_hll_face_flux": (None, [PD, D, PD]),
        "orc_bottom_friction": (None, [D, D, D, D, D, PD]),
        "orc_coriolis_force": (None, [D, D, D, PD]),
        "orc_wind_force": (None, [D, D, D, D, D, D, D, D, PD]),
        "orc_viscous_force": (I, [C.POINTER(A.swf_terrain), C.POINTER(A.swf_params), PD, PD, PD,
                                  I, I, PD]),
        "orc_surface_gradient_force": (I, [C.POINTER(A.swf_terrain), C.POINTER(A.swf_params), PD,
                                           PD, PD, I, I, PD]),
        "orc_total_volume": (D, [I, PD, D]),
        "orc_latitude_to_omega_z": (D, [D]),
    }
    optional = {"orc_face_fm"}  # the C restatement only (the reference keeps faces private)
    for name, (res, args) in sig.items():
        if name in optional and not hasattr(lib, name):
            continue
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


def load(kind: str = "orc"):
    """kind 'orc' (C restatement) or 'ref' (the real reference)."""
    if kind not in _libs:
        path = ORC_PATH if kind == "orc" else REF_PATH
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run oracle.pyorc.build())")
        _libs[kind] = _declare(C.CDLL(path))
    return _libs[kind]


def available(kind: str) -> bool:
    return os.path.exists(ORC_PATH if kind == "orc" else REF_PATH)


_ERR = {A.SWF_ECONFIG: ConfigError, A.SWF_ENUMERICAL: NumericalError, A.SWF_ERANGE: IndexError}


class OracleStepper:
    """Same surface as paper_1705_00614_b200.CsphTvdStepper, on the CPU checker."""

    def __init__(self, terrain, params, control, options=None, *, kind="orc"):
        options = options if options is not None else StepperOptions()
        self.lib = load(kind)
        self.kind = kind
        self._terrain, self._params, self._options = terrain, params, options
        m = Marshalled()
        t = m.terrain(terrain)
        p = m.params(params, terrain.nx * terrain.ny)
        k = m.control(control)
        o = m.options(options)
        ctx = C.c_void_p()
        rc = self.lib.orc_create(C.byref(t), C.byref(p), C.byref(k), C.byref(o), C.byref(ctx))
        self._raise(rc, None)
        self.ctx = ctx
        self.n = terrain.nx * terrain.ny

    def _raise(self, rc, ctx):
        if rc:
            msg = self.lib.orc_last_error(ctx)
            raise _ERR.get(rc, RuntimeError)(msg.decode() if msg else "")

    def _rc(self, rc):
        self._raise(rc, self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.orc_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_wind(self, wind):
        m = Marshalled()
        n, t, x, y = m.wind(wind)
        self._rc(self.lib.orc_set_wind(self.ctx, n, t, x, y))

    def set_sources(self, sources):
        m = Marshalled()
        arr = m.sources(sources)
        self._rc(self.lib.orc_set_sources(self.ctx, len(sources), arr))

    def set_control(self, control):
        k = Marshalled.control(control)
        self._rc(self.lib.orc_set_control(self.ctx, C.byref(k)))

    def set_options(self, options):
        o = Marshalled.options(options)
        self._options = options
        self._rc(self.lib.orc_set_options(self.ctx, C.byref(o)))

    def upload(self, state):
        self._rc(self.lib.orc_set_state(self.ctx, A.dptr(state.H), A.dptr(state.HUx),
                                        A.dptr(state.HUy), float(state.t)))

    def download(self, state):
        t = C.c_double()
        self._rc(self.lib.orc_get_state(self.ctx, A.dptr(state.H), A.dptr(state.HUx),
                                        A.dptr(state.HUy), C.byref(t)))
        state.t = t.value

    def step(self, state: FlowState, dt_cap: float = 0.0):
        self.upload(state)
        info = A.swf_step_info()
        rc = self.lib.orc_step(self.ctx, float(dt_cap), C.byref(info))
        self._rc(rc)
        self.download(state)
        return info_from_c(info)

    def run(self, n, dt_cap=0.0):
        done = C.c_int()
        info = A.swf_step_info()
        rc = self.lib.orc_run(self.ctx, int(n), float(dt_cap), C.byref(done), C.byref(info))
        self._rc(rc)
        return done.value, info_from_c(info)

    def _stage(self, sid, arg=0.0):
        tau = C.c_double(0.0)
        self._rc(self.lib.orc_stage(self.ctx, sid, float(arg), C.byref(tau)))
        return tau.value

    def begin_step(self, state):
        self.upload(state)
        self._stage(A.STAGE_BEGIN)

    def compute_forces(self, state):
        self._stage(A.STAGE_FORCES)

    def compute_dt(self, state, dt_cap=0.0):
        return self._stage(A.STAGE_DT, dt_cap)

    def predictor(self, state, tau):
        self._stage(A.STAGE_PREDICTOR, tau)

    def mid_forces(self, state, tau):
        self._stage(A.STAGE_MID_FORCES, tau)

    def corrector(self, state, tau):
        self._stage(A.STAGE_CORRECTOR, tau)

    def flux(self, state, tau):
        self._stage(A.STAGE_FLUX, tau)

    def final_update(self, state, tau):
        self._stage(A.STAGE_FINAL, tau)
        self.download(state)

    def scratch(self, name):
        out = np.empty(self.n)
        self._rc(self.lib.orc_scratch(self.ctx, A.SCRATCH_ID[name], A.dptr(out)))
        return out

    def face_fm(self, direction: int) -> np.ndarray:
        """fm of the x (0) or y (1) faces of the last flux stage (orc_face_fm)."""
        nx, ny = self._terrain.nx, self._terrain.ny
        n = (nx + 1) * ny if direction == 0 else nx * (ny + 1)
        out = np.empty(n)
        self._rc(self.lib.orc_face_fm(self.ctx, int(direction), A.dptr(out)))
        return out

    def mask(self):
        bs = self._options.block_size
        nbx = (self._terrain.nx + bs - 1) // bs
        nby = (self._terrain.ny + bs - 1) // bs
        inn = np.zeros(nbx * nby, np.int32)
        hal = np.zeros(nbx * nby, np.int32)
        a, b = C.c_int(), C.c_int()
        self._rc(self.lib.orc_mask(self.ctx, inn.ctypes.data_as(A.PI), hal.ctypes.data_as(A.PI),
                                   C.byref(a), C.byref(b)))
        return BlockMask(bs, a.value, b.value, self._terrain.nx, self._terrain.ny, inn, hal)

    def _volumes(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        self._rc(self.lib.orc_volumes(self.ctx, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def last_clamp_deficit(self):
        return self._volumes()[0]

    def last_source_volume(self):
        return self._volumes()[1]

    def last_boundary_outflow(self):
        return self._volumes()[2]
