"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/swf.h declares; with no GPU it fails loudly (no CPU
fallback)."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT, has_gpu


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "swf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(swf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_api():
    syms = declared_symbols()
    for s in ("swf_create", "swf_step", "swf_step_host", "swf_run", "swf_stage",
              "swf_download_scratch", "swf_strip_phase1", "swf_strip_phase2"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1705_00614_b200 import _lib
    lib = _lib.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_no_cpu_fallback_without_gpu():
    if has_gpu():
        pytest.skip("GPU present")
    from paper_1705_00614_b200 import CsphTvdStepper, scenarios
    sc = scenarios.dam_break_1d()
    with pytest.raises(RuntimeError, match="CUDA|device"):
        CsphTvdStepper(sc.terrain, sc.params, sc.control, sc.options)


def test_config_errors_before_device():
    """Validation happens on the host with the reference's messages even
    without a GPU (grid.cpp:13-21, stepper.cpp:31-37)."""
    import numpy as np
    from paper_1705_00614_b200 import (CsphTvdStepper, ConfigError, PhysicalParams, StepperOptions,
                                       Terrain, TimestepControl)
    T = Terrain(4, 4, 1.0, 0.0, 0.0, np.zeros(16))
    with pytest.raises(ConfigError, match="Courant"):
        CsphTvdStepper(T, PhysicalParams(), TimestepControl(courant=1.5))
    with pytest.raises(ConfigError, match="cell size"):
        CsphTvdStepper(Terrain(4, 4, 0.0, 0.0, 0.0, np.zeros(16)), PhysicalParams(), TimestepControl())
    b = np.zeros(16)
    b[3] = np.nan
    with pytest.raises(ConfigError, match="non-finite bed elevation at cell 3"):
        CsphTvdStepper(Terrain(4, 4, 1.0, 0.0, 0.0, b), PhysicalParams(), TimestepControl())
    with pytest.raises(ConfigError, match="block size"):
        CsphTvdStepper(T, PhysicalParams(), TimestepControl(), StepperOptions(block_size=0))
    with pytest.raises(ConfigError, match="nx and ny must be >= 1"):  # empty grid
        CsphTvdStepper(Terrain(0, 4, 1.0, 0.0, 0.0, np.zeros(0)), PhysicalParams(), TimestepControl())


def test_more_than_int32_cells_is_a_config_error():
    """The reference indexes cells with int (grid.hpp:27): grids above 2^31-1
    cells are rejected at creation, before any device or bed access."""
    import ctypes as C
    import numpy as np
    from paper_1705_00614_b200 import _abi as A
    from paper_1705_00614_b200._lib import lib
    L = lib()
    b = np.zeros(1)
    t = A.swf_terrain(50000, 50000, 1.0, 0.0, 0.0, A.dptr(b))
    p = A.swf_params(9.81, 0.02, 0.0, 0.0, 1e-3, 1.2, 1000.0, 1e-6, A.PD())
    k = A.swf_control(0.5, 10.0, 1e-9)
    o = A.swf_options(16, 1, 1, 0, 0, 0, 0)
    ctx = C.c_void_p()
    rc = L.swf_create(C.byref(t), C.byref(p), C.byref(k), C.byref(o), C.byref(ctx))
    assert rc == 1  # SWF_ECONFIG
    assert b"2^31-1" in L.swf_last_error(None)
