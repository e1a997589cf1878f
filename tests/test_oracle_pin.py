"""The CPU oracle (oracle/swf_oracle.c) pinned to the real reference:
golden vectors generated from the compiled reference (tests/golden), the
SPEC.md known answers, the glibc cbrt restatement, and — when the reference
compiles here — a stage-by-stage bitwise comparison of every scratch array."""
import ctypes as C
import math

import numpy as np
import pytest

from helpers import assert_bitwise, assert_state_bitwise, digest, golden, golden_factories, make
from paper_1705_00614_b200 import scenarios as S
from paper_1705_00614_b200 import _abi as A

G = golden()


@pytest.mark.parametrize("name", ["c1_dry_n002_capped", "c2_128", "flood64_all_physics", "lake128",
                                  "c1_dry_n0", "c1_wet_n002"])
def test_restatement_matches_golden(oracle_built, name):
    case = G["cases"][name]
    sc = golden_factories()[name]()
    o = make(oracle_built.OracleStepper, sc, kind="orc")
    st = sc.state.copy()
    info = None
    for _ in range(case["steps"]):
        info = o.step(st, case["dt_cap"])
    assert st.t.hex() == case["t"]
    assert digest(st) == case["sha256"]
    li = case["last_info"]
    assert info.tau.hex() == li["tau"]
    assert info.flux_blocks == li["flux_blocks"] and info.lagrangian_blocks == li["lagrangian_blocks"]
    assert info.clamp_deficit_volume.hex() == li["clamp_deficit_volume"]
    assert info.source_volume.hex() == li["source_volume"]
    assert info.boundary_outflow_volume.hex() == li["boundary_outflow_volume"]


def test_flood64_arrays(oracle_built):
    z = np.load(f"{oracle_built.HERE}/../tests/golden/flood64_all_physics.npz")
    sc = S.floodplain(64, 50.0)
    o = make(oracle_built.OracleStepper, sc, kind="orc")
    st = sc.state.copy()
    for _ in range(G["cases"]["flood64_all_physics"]["steps"]):
        o.step(st)
    assert_bitwise(st.H, z["H"], "H")
    assert_bitwise(st.HUx, z["HUx"], "HUx")
    assert_bitwise(st.HUy, z["HUy"], "HUy")


def test_spec_known_answers(oracle_built):
    """SPEC.md examples (§4 of SURVEY.md) on the restatement."""
    lib = oracle_built.load("orc")
    o2 = (C.c_double * 2)()
    lib.orc_bottom_friction(1.0, 0.0, 1.0, 9.81, 0.02, o2)
    assert o2[0] == pytest.approx(-3.924e-3, rel=1e-12) and o2[1] == 0.0
    assert [o2[0], o2[1]] == G["kat"]["friction"]
    lib.orc_coriolis_force(1.0, 0.0, 7.292e-5, o2)
    assert o2[1] == pytest.approx(-1.4584e-4, rel=1e-12) and [o2[0], o2[1]] == G["kat"]["coriolis"]
    lib.orc_wind_force(0.0, 0.0, 2.0, 5.0, 0.0, 1e-3, 1.2, 1000.0, o2)
    assert o2[0] == pytest.approx(1.5e-5, rel=1e-12) and [o2[0], o2[1]] == G["kat"]["wind"]
    o3 = (C.c_double * 3)()
    lib.orc_hll_face_flux((C.c_double * 6)(1.0, 0.0, 0.0, 0.0, 0.0, 0.0), 9.81, o3)
    # Ritter at x/t=0: H = 4/9, U = (2/3) sqrt(g)
    g = 9.81
    assert o3[0] == pytest.approx((4 / 9) * (2 / 3) * math.sqrt(g), rel=1e-12)
    assert [o3[0], o3[1], o3[2]] == G["kat"]["hll_dam_break"]
    lib.orc_hll_face_flux((C.c_double * 6)(2.0, 0.0, 0.0, 2.0, 0.0, 0.0), 9.81, o3)
    assert o3[0] == 0.0 and o3[1] == pytest.approx(0.5 * g * 4.0)
    assert lib.orc_latitude_to_omega_z(48.7) == G["kat"]["omega_48_7"]
    # total_volume
    H = np.ones(100)
    assert lib.orc_total_volume(100, A.dptr(H), 50.0) == 250000.0


def test_spec_viscous_and_gradient(oracle_built):
    lib = oracle_built.load("orc")
    from paper_1705_00614_b200._marshal import Marshalled
    from paper_1705_00614_b200.types import PhysicalParams, Terrain
    # viscous: nu=1, h=1, centre 0, four neighbours 1
    n = 3
    T = Terrain(n, n, 1.0, 0.0, 0.0, np.zeros(n * n))
    H = np.ones(n * n)
    HUx = np.zeros(n * n)
    HUx[[1, 3, 5, 7]] = 1.0
    HUy = np.zeros(n * n)
    m = Marshalled()
    t, p = m.terrain(T), m.params(PhysicalParams(nu=1.0), n * n)
    o2 = (C.c_double * 2)()
    assert lib.orc_viscous_force(C.byref(t), C.byref(p), A.dptr(H), A.dptr(HUx), A.dptr(HUy), 1, 1, o2) == 0
    assert (o2[0], o2[1]) == (4.0, 0.0)
    # gradient: eta rising 0.1 per 50 m in x
    T = Terrain(3, 1, 50.0, 0.0, 0.0, np.zeros(3))
    H = np.array([1.0, 1.1, 1.2])
    t = m.terrain(T)
    p = m.params(PhysicalParams(), 3)
    z = np.zeros(3)
    assert lib.orc_surface_gradient_force(C.byref(t), C.byref(p), A.dptr(H), A.dptr(z), A.dptr(z), 1, 0, o2) == 0
    assert o2[0] == pytest.approx(-0.01962, rel=1e-12)


def test_dt_known_answer(oracle_built):
    """H=1, h=50, K=0.5 -> 7.981886 s."""
    from paper_1705_00614_b200.types import (FlowState, PhysicalParams, StepperOptions, Terrain,
                                             TimestepControl)
    n = 4
    T = Terrain(n, n, 50.0, 0.0, 0.0, np.zeros(n * n))
    o = oracle_built.OracleStepper(T, PhysicalParams(n_manning=0.0), TimestepControl(), StepperOptions())
    st = FlowState(n, n, 0.0, np.ones(n * n), np.zeros(n * n), np.zeros(n * n))
    o.begin_step(st)
    o.compute_forces(st)
    assert o.compute_dt(st) == pytest.approx(0.5 * 50.0 / math.sqrt(9.81), rel=1e-15)
    assert round(o.compute_dt(st), 6) == 7.981886


def test_cbrt_restatement_matches_libm(oracle_built):
    """glibc s_cbrt.c restated == libm, bit for bit."""
    import hashlib
    lib = oracle_built.load("orc")
    rng = np.random.default_rng(1705)
    xs = np.concatenate([rng.uniform(0, 1e3, 50000), 2.0 ** rng.uniform(-60, 20, 50000),
                         -rng.uniform(0, 10, 1000)])
    ys = np.array([lib.orc_cbrt(float(x)) for x in xs])
    assert hashlib.sha256(ys.tobytes()).hexdigest() == G["kat"]["cbrt_sha256"]
    libm = C.CDLL("libm.so.6")
    libm.cbrt.restype = C.c_double
    libm.cbrt.argtypes = [C.c_double]
    extra = np.concatenate([2.0 ** rng.uniform(-1074, -1000, 2000), [0.0, -0.0, 1e-300, 5e-324,
                                                                     1.0, 8.0, 27.0, 1e308]])
    for x in extra:
        assert np.float64(lib.orc_cbrt(float(x))).view(np.int64) == np.float64(libm.cbrt(float(x))).view(np.int64), x


def _have_ref(pyorc):
    return pyorc.available("ref")


@pytest.mark.parametrize("skip", [True, False])
def test_stagewise_against_reference(oracle_built, skip):
    """Every scratch array after every stage, restatement vs real reference."""
    if not _have_ref(oracle_built):
        pytest.skip("reference not compiled here (no /root/reference)")
    sc = S.floodplain(96, 50.0)
    sc.options.skip_dry_blocks = skip
    a = make(oracle_built.OracleStepper, sc, kind="orc")
    b = make(oracle_built.OracleStepper, sc, kind="ref")
    sa, sb = sc.state.copy(), sc.state.copy()
    names = ["fn_fx", "fn_fy", "fn_fric_x", "fn_fric_y", "fn_sigma", "fm_fx", "fm_fy",
             "fm_fric_x", "fm_fric_y", "fm_sigma", "half_H", "Ht", "HVtx", "HVty", "drx", "dry",
             "Fh", "Fvx", "Fvy", "sigma", "src_vx", "src_vy"]
    for step in range(6):
        for o, s in ((a, sa), (b, sb)):
            o.begin_step(s)
            o.compute_forces(s)
        ta, tb = a.compute_dt(sa), b.compute_dt(sb)
        assert ta == tb
        for o, s in ((a, sa), (b, sb)):
            o.predictor(s, ta)
            o.mid_forces(s, ta)
            o.corrector(s, ta)
            o.flux(s, ta)
        for nm in names:
            assert_bitwise(a.scratch(nm), b.scratch(nm), f"step {step} {nm}")
        ma, mb = a.mask(), b.mask()
        assert np.array_equal(ma.interior_wet, mb.interior_wet) and np.array_equal(ma.halo_wet, mb.halo_wet)
        a.final_update(sa, ta)
        b.final_update(sb, tb)
        assert_state_bitwise(sa, sb, f"step {step}")
        assert a._volumes() == b._volumes()
