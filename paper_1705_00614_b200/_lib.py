"""Loader for the in-tree CUDA library libswflood_cuda.so (the product path).

There is deliberately no fallback: if the library is missing or no CUDA
device is usable, calls fail loudly (ImportError / SWF_ECUDA).
"""
import ctypes as C
import os

from . import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
# SWF_FLAVOR=fast selects the opt-in FAST build (libswflood_cuda_fast.so);
# SWF_LIB names any build explicitly (developer A/B variants)
LIB_PATH = os.environ.get("SWF_LIB") or os.path.join(
    HERE, "libswflood_cuda_fast.so" if os.environ.get("SWF_FLAVOR") == "fast"
    else "libswflood_cuda.so")

_lib = None


def _sig(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)


def declare(lib):
    P, I, D, V = C.c_void_p, C.c_int, C.c_double, None
    PD, PI = A.PD, A.PI
    PT = C.POINTER(A.swf_terrain)
    PP = C.POINTER(A.swf_params)
    PK = C.POINTER(A.swf_control)
    PO = C.POINTER(A.swf_options)
    PS = C.POINTER(A.swf_source)
    PN = C.POINTER(A.swf_step_info)
    PPD = C.POINTER(PD)
    _sig(lib, "swf_create", I, PT, PP, PK, PO, C.POINTER(P))
    _sig(lib, "swf_create_strip", I, PT, PP, PK, PO, I, I, I, C.POINTER(P))
    _sig(lib, "swf_destroy", V, P)
    _sig(lib, "swf_last_error", C.c_char_p, P)
    _sig(lib, "swf_set_wind", I, P, I, PD, PD, PD)
    _sig(lib, "swf_set_sources", I, P, I, PS)
    _sig(lib, "swf_set_control", I, P, PK)
    _sig(lib, "swf_get_control", I, P, PK)
    _sig(lib, "swf_set_options", I, P, PO)
    _sig(lib, "swf_get_options", I, P, PO)
    _sig(lib, "swf_upload_state", I, P, PD, PD, PD, D)
    _sig(lib, "swf_download_state", I, P, PD, PD, PD, PD)
    _sig(lib, "swf_device_state", I, P, PPD, PPD, PPD)
    _sig(lib, "swf_step_host", I, P, PD, PD, PD, PD, D, PN)
    _sig(lib, "swf_step", I, P, D, PN)
    _sig(lib, "swf_run", I, P, I, D, PI, PN)
    _sig(lib, "swf_sync", I, P)
    _sig(lib, "swf_active_tiles", I, P, PI, PI, PI)
    _sig(lib, "swf_set_timing", I, P, I)
    _sig(lib, "swf_timing_read", I, P, I, PD)
    _sig(lib, "swf_stream", P, P)
    _sig(lib, "swf_set_mode", I, P, I)
    _sig(lib, "swf_stage", I, P, I, D, PD)
    _sig(lib, "swf_download_scratch", I, P, I, PD)
    _sig(lib, "swf_download_mask", I, P, PI, PI, PI, PI)
    _sig(lib, "swf_last_volumes", I, P, PD, PD, PD)
    _sig(lib, "swf_dev_hll_face_flux", I, I, PD, D, PD)
    _sig(lib, "swf_dev_cbrt", I, I, PD, PD)
    _sig(lib, "swf_dev_rdiv", I, I, PD, PD)
    _sig(lib, "swf_dev_rdiv_spec", I, I, PD, PD)
    _sig(lib, "swf_dev_sqrt_spec", I, I, PD, PD)
    _sig(lib, "swf_dev_bottom_friction", I, I, PD, D, D, PD)
    _sig(lib, "swf_strip_phase1", I, P, D, PD)
    _sig(lib, "swf_strip_phase2", I, P, D, D, PN)
    _sig(lib, "swf_strip_halo_ptrs", I, P, I, PPD, PPD, C.POINTER(C.c_size_t))
    _sig(lib, "swf_strip_rows", I, P, PI, PI, PI, PI)
    _sig(lib, "swf_strip_pack", I, P, I, C.c_void_p)
    _sig(lib, "swf_strip_unpack", I, P, I, C.c_void_p)
    _sig(lib, "swf_last_ingest_bytes", I, P, C.POINTER(C.c_longlong))
    _sig(lib, "swf_last_writeback_bytes", I, P, C.POINTER(C.c_longlong))
    _sig(lib, "swf_set_host_mirror", I, P, I)
    _sig(lib, "swf_build_flavor", C.c_char_p)
    _sig(lib, "swf_host_changed", I, P)
    _sig(lib, "swf_debug_redo_counts", I, P, PI)
    _sig(lib, "swf_debug_region_loads", I, P)
    _sig(lib, "swf_device_buffers", I, P, C.POINTER(C.c_void_p))
    _sig(lib, "swf_strip_set_peer", I, P, I, C.POINTER(C.c_void_p), I)
    _sig(lib, "swf_strip_begin_batch", I, P)
    _sig(lib, "swf_strip_forces", I, P, D, I)
    _sig(lib, "swf_strip_local_speed", I, P, C.c_void_p)
    _sig(lib, "swf_strip_finish", I, P, C.c_void_p, D)
    _sig(lib, "swf_strip_end_batch", I, P, PI, PN)
    _sig(lib, "swf_strip_settle", I, P, I)
    _sig(lib, "swf_group_create", I, C.POINTER(P), I, C.POINTER(P))
    _sig(lib, "swf_group_run", I, P, I, D, PI, PN)
    _sig(lib, "swf_group_last_error", C.c_char_p, P)
    _sig(lib, "swf_group_destroy", V, P)
    _sig(lib, "swf_strip_steps_done", I, P)
    _sig(lib, "swf_strip_host_phase1", I, P, C.c_void_p, C.c_void_p, C.c_void_p, PD, D, PD)
    _sig(lib, "swf_strip_host_phase2", I, P, C.c_void_p, C.c_void_p, C.c_void_p, PD, D, D, PN)
    _sig(lib, "swf_strip_pack_async", I, P, I, C.c_void_p)
    _sig(lib, "swf_strip_unpack_async", I, P, I, C.c_void_p)
    PND = C.POINTER(A.swf_nest_desc)
    _sig(lib, "swf_nest_create", I, P, P, PND, C.POINTER(P))
    _sig(lib, "swf_nest_destroy", V, P)
    _sig(lib, "swf_nest_last_error", C.c_char_p, P)
    _sig(lib, "swf_nest_ghost_count", I, P, C.POINTER(C.c_size_t))
    _sig(lib, "swf_nest_prolong", I, P, I)
    _sig(lib, "swf_nest_apply_ghosts", I, P, D)
    _sig(lib, "swf_nest_restrict", I, P)
    _sig(lib, "swf_nest_download_ghosts", I, P, I, PD)
    _sig(lib, "swf_coupled_step", I, P, C.POINTER(P), I, D, C.POINTER(A.swf_coupled_info))
    return lib


def lib():
    """The loaded CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        _lib = declare(C.CDLL(LIB_PATH))
    return _lib
