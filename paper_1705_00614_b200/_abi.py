"""ctypes mirror of the C ABI in include/swf.h (the drop-in boundary).

The struct layouts here must match include/swf.h byte for byte; both the
product library (libswflood_cuda.so) and the test-only checker libraries
(oracle/liborc.so, oracle/_ref/libswflood_ref.so) take these structs.
"""
import ctypes as C

SWF_OK, SWF_ECONFIG, SWF_ENUMERICAL, SWF_ERANGE, SWF_ECUDA = 0, 1, 2, 3, 4
EDGE_REFLECTIVE, EDGE_OPEN = 0, 1
SOURCE_DISCHARGE, SOURCE_RAIN = 0, 1

(STAGE_BEGIN, STAGE_FORCES, STAGE_DT, STAGE_PREDICTOR, STAGE_MID_FORCES,
 STAGE_CORRECTOR, STAGE_FLUX, STAGE_FINAL) = range(8)

SCRATCH = [
    "fn_fx", "fn_fy", "fn_fric_x", "fn_fric_y", "fn_sigma",
    "fm_fx", "fm_fy", "fm_fric_x", "fm_fric_y", "fm_sigma",
    "half_H", "half_HUx", "half_HUy",
    "Ht", "HVtx", "HVty",
    "drx", "dry",
    "Fh", "Fvx", "Fvy",
    "sigma", "src_vx", "src_vy",
]
SCRATCH_ID = {name: i for i, name in enumerate(SCRATCH)}

PD = C.POINTER(C.c_double)
PI = C.POINTER(C.c_int)


class swf_terrain(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("h", C.c_double),
                ("x0", C.c_double), ("y0", C.c_double), ("b", PD)]


class swf_params(C.Structure):
    _fields_ = [("g", C.c_double), ("n_manning", C.c_double), ("nu", C.c_double),
                ("omega_z", C.c_double), ("c_a", C.c_double), ("rho_air", C.c_double),
                ("rho_water", C.c_double), ("eps_dry", C.c_double), ("n_field", PD)]


class swf_control(C.Structure):
    _fields_ = [("courant", C.c_double), ("dt_max", C.c_double), ("dt_min", C.c_double)]


class swf_options(C.Structure):
    _fields_ = [("block_size", C.c_int), ("skip_dry_blocks", C.c_int), ("workers", C.c_int),
                ("west", C.c_int), ("east", C.c_int), ("south", C.c_int), ("north", C.c_int)]


class swf_source(C.Structure):
    _fields_ = [("kind", C.c_int), ("i0", C.c_int), ("j0", C.c_int), ("i1", C.c_int),
                ("j1", C.c_int), ("n_hydro", C.c_int), ("hydro_t", PD), ("hydro_q", PD),
                ("rate", C.c_double), ("vx", C.c_double), ("vy", C.c_double)]


class swf_step_info(C.Structure):
    _fields_ = [("tau", C.c_double), ("active_fraction", C.c_double),
                ("lagrangian_blocks", C.c_int), ("flux_blocks", C.c_int),
                ("total_blocks", C.c_int), ("timings", C.c_double * 8),
                ("clamp_deficit_volume", C.c_double), ("source_volume", C.c_double),
                ("boundary_outflow_volume", C.c_double)]


def dptr(a):
    """double* of a C-contiguous float64 numpy array (or NULL for None)."""
    if a is None:
        return PD()
    assert a.dtype.name == "float64" and a.flags["C_CONTIGUOUS"], "need C-contiguous float64"
    return a.ctypes.data_as(PD)


class swf_nest_desc(C.Structure):
    _fields_ = [("i0", C.c_int), ("j0", C.c_int), ("ni", C.c_int), ("nj", C.c_int),
                ("r", C.c_int), ("ghost", C.c_int), ("two_way", C.c_int)]


class swf_coupled_info(C.Structure):
    _fields_ = [("tau", C.c_double), ("substeps_total", C.c_int), ("substeps_max", C.c_int),
                ("fine_tau_min", C.c_double), ("coarse", swf_step_info),
                ("reflux_clamp_volume", C.c_double)]
