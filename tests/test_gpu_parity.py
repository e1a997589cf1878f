"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the golden vectors generated from the compiled reference.  The bar is
bit-exact equality of H, HUx, HUy, t and tau (fp64, no tolerance), which
also makes the wet/dry mask bit-exact."""
import ctypes as C
import hashlib

import numpy as np
import pytest

from helpers import (assert_bitwise, assert_state_bitwise, digest, golden, golden_factories, make)
from paper_1705_00614_b200 import scenarios as S
from paper_1705_00614_b200.types import HydrographSample as HS

pytestmark = pytest.mark.gpu
G = golden()


@pytest.fixture(scope="module")
def gpu_cls():
    from paper_1705_00614_b200 import CsphTvdStepper
    return CsphTvdStepper


# ---------------------------------------------------------------- device KATs

def test_device_cbrt_matches_glibc(oracle_built):
    from paper_1705_00614_b200.stepper import cbrt_device
    rng = np.random.default_rng(1705)
    xs = np.concatenate([rng.uniform(0, 1e3, 50000), 2.0 ** rng.uniform(-60, 20, 50000),
                         -rng.uniform(0, 10, 1000)])
    ys = cbrt_device(xs)
    assert hashlib.sha256(ys.tobytes()).hexdigest() == G["kat"]["cbrt_sha256"]
    lib = oracle_built.load("orc")
    more = np.concatenate([2.0 ** rng.uniform(-1074, 1023, 20000), rng.uniform(1e-7, 30, 20000),
                           [0.0, -0.0, 5e-324, 1e-300, 1.0, 8.0, 27.0, 1e308]])
    got = cbrt_device(more)
    exp = np.array([lib.orc_cbrt(float(x)) for x in more])
    assert_bitwise(got, exp, "cbrt")


def test_device_hll_matches_oracle(oracle_built):
    from paper_1705_00614_b200.stepper import hll_face_flux_device
    rng = np.random.default_rng(7)
    n = 200000
    x = np.column_stack([rng.uniform(0, 5, n), rng.normal(0, 3, n), rng.normal(0, 1, n),
                         rng.uniform(0, 5, n), rng.normal(0, 3, n), rng.normal(0, 1, n)])
    x[: n // 4, 0] = 0.0  # dry left
    x[n // 4: n // 2, 3] = 0.0  # dry right
    x[n // 2: n // 2 + 100, [0, 3]] = 0.0  # dry/dry
    e = slice(n // 2 + 100, n // 2 + 40000)  # depths around the dry threshold
    x[e, 0] = rng.uniform(0, 3e-6, e.stop - e.start)
    x[e, 3] = rng.uniform(0, 3e-6, e.stop - e.start)
    w = slice(n // 2 + 40000, n // 2 + 60000)  # wide dynamic range
    x[w, 0] = 10.0 ** rng.uniform(-8, 3, w.stop - w.start)
    x[w, 1] = rng.normal(0, 1, w.stop - w.start) * 10.0 ** rng.uniform(-6, 2, w.stop - w.start)
    got = hll_face_flux_device(x, 9.81)
    lib = oracle_built.load("orc")
    o3 = (C.c_double * 3)()
    exp = np.empty_like(got)
    for k in range(n):
        lib.orc_hll_face_flux((C.c_double * 6)(*x[k]), 9.81, o3)
        exp[k] = o3[:]
    assert_bitwise(got, exp, "hll")
    assert list(hll_face_flux_device(np.array([[1.0, 0, 0, 0, 0, 0]]), 9.81)[0]) == G["kat"]["hll_dam_break"]


def test_device_rdiv_matches_division():
    """The shared-reciprocal division used by the kernels is bit-identical to
    nvcc's IEEE division on random, extreme and special operands."""
    from paper_1705_00614_b200._lib import lib
    from paper_1705_00614_b200 import _abi as A
    rng = np.random.default_rng(11)
    n = 400000
    a = np.concatenate([rng.normal(0, 1, n) * 10.0 ** rng.integers(-30, 30, n),
                        2.0 ** rng.uniform(-1074, 1023, n) * rng.choice([-1, 1], n),
                        rng.uniform(-5, 5, n)])
    b = np.concatenate([rng.normal(0, 1, n) * 10.0 ** rng.integers(-30, 30, n),
                        2.0 ** rng.uniform(-1074, 1023, n) * rng.choice([-1, 1], n),
                        rng.uniform(0.4, 1.6, n) * 50.0])
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
                        1.7976931348623157e308, 1.0, -1.0, 3.0])
    sa, sb = np.meshgrid(special, special)
    a = np.concatenate([a, sa.ravel()])
    b = np.concatenate([b, sb.ravel()])
    ab = np.ascontiguousarray(np.column_stack([a, b]))
    out = np.empty_like(ab)
    assert lib().swf_dev_rdiv(ab.shape[0], A.dptr(ab), A.dptr(out)) == 0
    assert_bitwise(out[:, 0], out[:, 1], "rdiv vs a/b")
    with np.errstate(all="ignore"):
        assert_bitwise(out[:, 1], a / b, "device a/b vs IEEE")
    # the speculative form: every ACCEPTED quotient is the IEEE one; zeros over
    # finite non-zero divisors are accepted, tiny/denormal operands are not
    spec = np.empty_like(ab)
    assert lib().swf_dev_rdiv_spec(ab.shape[0], A.dptr(ab), A.dptr(spec)) == 0
    acc = spec[:, 1] == 1.0
    with np.errstate(all="ignore"):
        q = a / b
    assert_bitwise(spec[acc, 0], q[acc], "accepted speculative quotient vs a/b")
    assert acc.mean() > 0.6
    z = (a == 0) & (np.abs(b) > 2.0 ** -1000) & (np.abs(b) < 2.0 ** 1000)
    assert acc[z].all()


def test_device_sqrt_spec():
    """The kernels' square root (speculative when built with SWF_SPEC_SQRT):
    every accepted result is the IEEE sqrt bit for bit; zeros and normal
    operands are accepted, tiny/denormal/negative/special ones are not."""
    from paper_1705_00614_b200._lib import lib
    from paper_1705_00614_b200 import _abi as A
    rng = np.random.default_rng(12)
    n = 400000
    x = np.concatenate([2.0 ** rng.uniform(-1074, 1024, n),
                        rng.uniform(0, 1e4, n), rng.uniform(0.5, 2.0, n),
                        np.nextafter(2.0 ** rng.integers(-1022, 1023, n), np.inf),
                        -rng.uniform(0, 10, 1000),
                        [0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 2.0 ** -970,
                         np.nextafter(2.0 ** -970, 0), 1.7976931348623157e308, 1.0, 4.0]])
    out = np.empty((x.size, 2))
    assert lib().swf_dev_sqrt_spec(x.size, A.dptr(x), A.dptr(out)) == 0
    acc = out[:, 1] == 1.0
    with np.errstate(all="ignore"):
        ref = np.sqrt(x)
    assert_bitwise(out[acc, 0], ref[acc], "accepted sqrt vs IEEE")
    normal = (x >= 2.0 ** -970) & np.isfinite(x)
    assert acc[normal].all() and acc[x == 0].all()


def test_device_friction_known_answer():
    from paper_1705_00614_b200.stepper import bottom_friction_device
    f = bottom_friction_device(np.array([[1.0, 0.0]]), np.array([1.0]), 9.81, 0.02)
    assert list(f[0]) == G["kat"]["friction"]


# ------------------------------------------------------- full-step golden runs

@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("name", list(G["cases"].keys()))
def test_golden_case(gpu_cls, name, mode):
    case = G["cases"][name]
    sc = golden_factories()[name]()
    s = make(gpu_cls, sc, mode=mode)
    st = sc.state.copy()
    s.upload(st)
    info = None
    for _ in range(case["steps"]):
        info = s.step_resident(case["dt_cap"])
    s.download(st)
    assert st.t.hex() == case["t"], (st.t, float.fromhex(case["t"]))
    assert digest(st) == case["sha256"]
    li = case["last_info"]
    assert info.tau.hex() == li["tau"]
    assert info.lagrangian_blocks == li["lagrangian_blocks"]
    assert info.flux_blocks == li["flux_blocks"]
    assert info.total_blocks == li["total_blocks"]
    assert info.active_fraction.hex() == li["active_fraction"]
    # both paths sum the diagnostics in the reference's order (the stage path
    # per block; the fused path from the terms k_step stores, fused_exact_volumes)
    assert info.clamp_deficit_volume.hex() == li["clamp_deficit_volume"]
    assert info.source_volume.hex() == li["source_volume"]
    assert info.boundary_outflow_volume.hex() == li["boundary_outflow_volume"]


def test_flood64_arrays_and_host_step(gpu_cls):
    """The drop-in host-buffer step() against the golden arrays."""
    z = np.load(f"{__file__.rsplit('/', 1)[0]}/golden/flood64_all_physics.npz")
    sc = S.floodplain(64, 50.0)
    s = make(gpu_cls, sc)
    st = sc.state.copy()
    for _ in range(G["cases"]["flood64_all_physics"]["steps"]):
        s.step(st)
    assert_bitwise(st.H, z["H"], "H")
    assert_bitwise(st.HUx, z["HUx"], "HUx")
    assert_bitwise(st.HUy, z["HUy"], "HUy")
    assert st.t == float(z["t"][0])


def test_host_step_pinned_write_back(gpu_cls, oracle_built):
    """step() on pinned host arrays writes back only the updated tiles from
    the kernel; the result must still be the full new state."""
    import torch
    sc = S.floodplain(16384, 50.0, window=(7600, 7000, 333, 250))
    pin = lambda a: torch.from_numpy(a.copy()).pin_memory().numpy()
    st = sc.state.copy()
    st.H, st.HUx, st.HUy = pin(st.H), pin(st.HUx), pin(st.HUy)
    so = sc.state.copy()
    g = make(gpu_cls, sc)
    o = make(oracle_built.OracleStepper, sc, kind="orc")
    for _ in range(12):
        ig, io = g.step(st), o.step(so)
        assert ig.tau == io.tau
    assert_state_bitwise(st, so, "pinned host step")


# ------------------------------------------------------------ stage API parity

def _kind(oracle_built, kind):
    """'orc' = the C restatement; 'ref' = the REAL reference compiled from
    /root/reference (oracle/_ref/libswflood_ref.so, which travels to the GPU
    box with the snapshot) -- compared directly, not through the restatement."""
    if kind == "ref" and not oracle_built.available("ref"):
        pytest.skip("the compiled reference (oracle/_ref) is not present")
    return kind


@pytest.mark.parametrize("kind", ["orc", "ref"])
@pytest.mark.parametrize("skip", [True, False])
def test_stagewise_against_oracle(gpu_cls, oracle_built, skip, kind):
    sc = S.floodplain(96, 50.0)
    sc.options.skip_dry_blocks = skip
    a = make(oracle_built.OracleStepper, sc, kind=_kind(oracle_built, kind))
    b = make(gpu_cls, sc)
    sa, sb = sc.state.copy(), sc.state.copy()
    names = ["fn_fx", "fn_fy", "fn_fric_x", "fn_fric_y", "fn_sigma", "fm_fx", "fm_fy",
             "fm_fric_x", "fm_fric_y", "fm_sigma", "half_H", "half_HUx", "half_HUy", "Ht",
             "HVtx", "HVty", "drx", "dry", "Fh", "Fvx", "Fvy", "sigma", "src_vx", "src_vy"]
    if kind == "ref":  # the reference's accessors (stepper.hpp:102-119) have no half momenta
        names = [nm for nm in names if nm not in ("half_HUx", "half_HUy")]
    for step in range(5):
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
            assert_bitwise(b.scratch(nm), a.scratch(nm), f"step {step} {nm}")
        ma, mb = a.mask(), b.mask()
        assert np.array_equal(ma.interior_wet, mb.interior_wet)
        assert np.array_equal(ma.halo_wet, mb.halo_wet)
        a.final_update(sa, ta)
        b.final_update(sb, tb)
        assert_state_bitwise(sb, sa, f"step {step}")
        assert b._volumes() == a._volumes()


# ----------------------------------------------------------- properties

def test_run_equals_repeated_step(gpu_cls):
    sc = S.floodplain(200, 50.0)
    a, b = make(gpu_cls, sc), make(gpu_cls, sc)
    sa, sb = sc.state.copy(), sc.state.copy()
    a.upload(sa)
    b.upload(sb)
    done, _ = a.run(23)
    assert done == 23
    for _ in range(23):
        b.step_resident()
    a.download(sa)
    b.download(sb)
    assert_state_bitwise(sa, sb, "run vs step")


@pytest.mark.parametrize("bs", [7, 16, 32])
def test_skip_and_block_size_equivalence(gpu_cls, bs):
    """skipping on vs off, any block size -> identical bits."""
    sc = S.circular_dam_break(512, 8.0, 64)
    ref = make(gpu_cls, sc)
    st_ref = sc.state.copy()
    ref.options().skip_dry_blocks = False
    ref.upload(st_ref)
    ref.run(40)
    ref.download(st_ref)
    sc.options.block_size = bs
    s = make(gpu_cls, sc)
    st = sc.state.copy()
    s.upload(st)
    s.run(40)
    s.download(st)
    assert_state_bitwise(st, st_ref, f"B={bs}")


@pytest.mark.parametrize("kind", ["orc", "ref"])
def test_medium_floodplain_vs_oracle(gpu_cls, oracle_built, kind):
    sc = S.floodplain(16384, 50.0, window=(7000, 7600, 300, 260))  # a crop of C3
    a = make(oracle_built.OracleStepper, sc, kind=_kind(oracle_built, kind))
    b = make(gpu_cls, sc)
    sa, sb = sc.state.copy(), sc.state.copy()
    for _ in range(8):
        ia, ib = a.step(sa), b.step(sb)
        assert ia.tau == ib.tau
    assert_state_bitwise(sb, sa, "C3 crop")


def test_lake_at_rest_is_fixed_point(gpu_cls):
    sc = S.lake_at_rest(128)
    s = make(gpu_cls, sc)
    st = sc.state.copy()
    s.upload(st)
    s.run(1000)
    s.download(st)
    u = np.where(st.H > 1e-6, np.hypot(st.HUx, st.HUy) / np.maximum(st.H, 1e-300), 0.0)
    assert u.max() <= 1e-10
    assert np.abs(st.H - sc.state.H).max() <= 1e-12


def test_mass_conservation_closed_basin(gpu_cls):
    sc = S.circular_dam_break(1024, 8.0, 128, n_manning=0.03)
    s = make(gpu_cls, sc)
    st = sc.state.copy()
    v0 = st.H.sum()
    s.upload(st)
    s.run(300)
    s.download(st)
    assert abs(st.H.sum() - v0) / v0 < 1e-12


# ------------------------------------------------------------- error paths

def _cfl_case():
    """A drain that empties a moving cell to ~1 mm within the half step makes
    u_1/2 = q/H_1/2 explode, so |dr| >= h/2 (stepper.cpp:378-380)."""
    from paper_1705_00614_b200.types import CellRect, HydrographSample, SourceKind, SourceSpec
    sc = S.dam_break_1d(True, 0.0, nx=64, ny=16)
    sc.state.H[:] = 1.0
    sc.state.HUx[:] = 1.0
    sig = -2.0 * (1.0 - 1e-3) / 0.1
    sc.sources = [SourceSpec(SourceKind.Discharge, "drain", CellRect(40, 5, 40, 5),
                             [HydrographSample(0.0, sig)])]
    return sc


def test_cfl_abort_leaves_state_untouched(gpu_cls, oracle_built):
    from paper_1705_00614_b200 import NumericalError
    sc = _cfl_case()
    for mode in (0, 1):
        s = make(gpu_cls, sc, mode=mode)
        o = make(oracle_built.OracleStepper, sc, kind="orc")
        st, so = sc.state.copy(), sc.state.copy()
        with pytest.raises(NumericalError) as eo:
            o.step(so, 0.1)
        before = st.copy()
        with pytest.raises(NumericalError) as eg:
            s.step(st, 0.1)
        assert str(eg.value) == str(eo.value)
        assert "particle displacement reached h/2 at cell (40,5)" in str(eg.value)
        assert_state_bitwise(st, before, "state changed on abort")


def test_long_run_after_an_early_abort_stays_clean(gpu_cls, oracle_built):
    """swf_run enqueues all its steps up front: after a CFL abort in the first
    step, the remaining 300 steps of the run are stopped on the device.  They
    must neither grow the work lists nor rewrite the tile flags, so the state
    is untouched and the same context then steps another state bit for bit."""
    from paper_1705_00614_b200 import NumericalError
    sc = _cfl_case()
    sc.control.dt_max = 0.1  # tau = 0.1 (the failing step of test_cfl_abort_...)
    s = make(gpu_cls, sc)
    st = sc.state.copy()
    s.upload(st)
    with pytest.raises(NumericalError, match="particle displacement"):
        s.run(301)
    after = sc.state.copy()
    s.download(after)
    assert_state_bitwise(after, sc.state, "state after the aborted run")
    # the same context, a healthy state: bitwise against the oracle
    good = sc.state.copy()
    good.HUx[:] = 0.1
    o = make(oracle_built.OracleStepper, sc, kind="orc")
    ref = good.copy()
    s.upload(good)
    s.run(40, 0.01)
    s.download(good)
    for _ in range(40):
        o.step(ref, 0.01)
    assert_state_bitwise(good, ref, "steps after the aborted run")


def test_dt_floor_abort(gpu_cls):
    from paper_1705_00614_b200 import NumericalError
    sc = S.dam_break_1d(False, 0.0, nx=64, ny=8)
    sc.control.dt_min = 5.0
    sc.control.dt_max = 10.0
    s = make(gpu_cls, sc)
    st = sc.state.copy()
    before = st.copy()
    with pytest.raises(NumericalError, match="fell below the abort floor"):
        s.step(st)
    assert_state_bitwise(st, before)


def test_run_stops_at_failure(gpu_cls):
    from paper_1705_00614_b200 import NumericalError
    sc = _cfl_case()
    sc.sources[0].hydrograph = [HS(0.0, 0.0), HS(2.0, 0.0), HS(2.05, -19.98)]
    a = make(gpu_cls, sc)
    st = sc.state.copy()
    n_ok = 0
    for _ in range(200):
        try:
            a.step(st, 0.1)
            n_ok += 1
        except NumericalError:
            break
    assert 0 < n_ok < 200
    b = make(gpu_cls, sc)
    sb = sc.state.copy()
    b.upload(sb)
    with pytest.raises(NumericalError):
        b.run(200, 0.1)
    b.download(sb)
    assert_state_bitwise(sb, st, "run() state after failure")


def test_pinned_host_step_sparse_ingest_matches_oracle(gpu_cls, oracle_built):
    """step(FlowState) on PINNED arrays: depth copied in full, momentum read
    over PCIe for the flux-active tiles only, updated tiles written back in
    place.  Bit-identical to the oracle, including junk momentum in dry cells
    the step must neither read nor overwrite."""
    import torch
    from paper_1705_00614_b200.types import ConfigError, FlowState
    sc = S.floodplain(256, 50.0)
    st = sc.state.copy()
    rng = np.random.default_rng(5)
    dry = st.H <= sc.params.eps_dry
    st.HUx[dry] = rng.normal(0, 1, dry.sum())  # never read by the reference for dry cells...
    st.HUy[dry] = rng.normal(0, 1, dry.sum())
    pin = lambda a: torch.from_numpy(a.copy()).pin_memory().numpy()
    hs = FlowState(st.nx, st.ny, 0.0, pin(st.H), pin(st.HUx), pin(st.HUy))
    cpu_state = st.copy()
    g = make(gpu_cls, sc)
    o = make(oracle_built.OracleStepper, sc)
    for k in range(12):
        ia = g.step(hs)
        ib = o.step(cpu_state)
        assert ia.tau == ib.tau, k
        assert g.last_ingest_bytes() < 3 * 8 * st.H.size
    assert_state_bitwise(hs, cpu_state, "pinned sparse ingest")
    with pytest.raises(ConfigError, match="upload"):
        g.download(FlowState(st.nx, st.ny, 0.0, np.empty_like(st.H), np.empty_like(st.H),
                             np.empty_like(st.H)))
    g.upload(hs)  # a fresh upload makes the resident state complete again
    g.step_resident()
    o.step(cpu_state)
    out = FlowState(st.nx, st.ny, 0.0, np.empty_like(st.H), np.empty_like(st.H), np.empty_like(st.H))
    g.download(out)
    assert_state_bitwise(out, cpu_state, "resident after pinned steps")


def test_pinned_host_steps_follow_host_side_edits(gpu_cls, oracle_built):
    """Between pinned host steps the caller edits its arrays anywhere: a
    puddle poured on dry ground far from the flood, a wet patch drained.  The
    forces phase of a host step visits only the tiles the fresh block mask
    flags, so new water must be seen there and drained tiles skipped; state,
    tau and the block counts stay identical to the oracle."""
    import torch
    from paper_1705_00614_b200.types import FlowState
    sc = S.floodplain(256, 50.0)
    st = sc.state.copy()
    pin = lambda a: torch.from_numpy(a.copy()).pin_memory().numpy()
    hs = FlowState(st.nx, st.ny, 0.0, pin(st.H), pin(st.HUx), pin(st.HUy))
    cpu_state = st.copy()
    g = make(gpu_cls, sc)
    o = make(oracle_built.OracleStepper, sc)
    H2 = hs.H.reshape(st.ny, st.nx)
    dry = np.argwhere(H2 <= sc.params.eps_dry)
    wet = np.argwhere(H2 > sc.params.eps_dry)
    assert len(dry) and len(wet)
    for k in range(8):
        if k == 2:  # a puddle on dry ground (a 3x3 patch around a dry cell)
            j, i = dry[len(dry) // 3]
            for a in (hs, cpu_state):
                a.H.reshape(st.ny, st.nx)[max(j - 1, 0):j + 2, max(i - 1, 0):i + 2] += 0.5
        if k == 5:  # drain a wet patch
            j, i = wet[len(wet) // 2]
            for a in (hs, cpu_state):
                sl = (slice(max(j - 8, 0), j + 8), slice(max(i - 8, 0), i + 8))
                a.H.reshape(st.ny, st.nx)[sl] = 0.0
                a.HUx.reshape(st.ny, st.nx)[sl] = 0.0
                a.HUy.reshape(st.ny, st.nx)[sl] = 0.0
        ia = g.step(hs)
        ib = o.step(cpu_state)
        assert ia.tau == ib.tau, k
        assert (ia.lagrangian_blocks, ia.flux_blocks) == (ib.lagrangian_blocks, ib.flux_blocks), k
    assert_state_bitwise(hs, cpu_state, "pinned steps with host-side edits")


@pytest.mark.parametrize("case,bs,skip", [("flood256", 16, True), ("flood256", 7, True),
                                          ("flood256", 16, False), ("c2", 16, True),
                                          ("c1_dry", 32, True)])
def test_step_info_volumes_bitwise_every_step(gpu_cls, oracle_built, case, bs, skip):
    """StepInfo's clamp deficit, source volume and boundary outflow of the
    fused path, every step, bit for bit the reference's serial sums
    (final_update, stepper.cpp:676-701), for block sizes that do and do not
    align with the 32 x 16 tiles and with skipping on and off."""
    from paper_1705_00614_b200.types import CellRect, SourceKind, SourceSpec, Vec2
    if case == "flood256":  # + a drain strong enough to empty its cells (clamped Ht)
        sc = S.floodplain(256, 50.0)
        sc.sources.append(SourceSpec(SourceKind.Discharge, "drain2", CellRect(40, 127, 46, 133),
                                     [HS(0.0, -5e4)], 0.0, Vec2(0.0, 0.0)))
    elif case == "c2":
        sc = S.circular_dam_break(256, 8.0, 40, n_manning=0.03)
    else:
        sc = S.dam_break_1d(False, 0.02)
    sc.options.block_size = bs
    sc.options.skip_dry_blocks = skip
    g = make(gpu_cls, sc)
    o = make(oracle_built.OracleStepper, sc)
    st = sc.state.copy()
    g.upload(st)
    ref = sc.state.copy()
    nonzero = [0, 0, 0]
    for k in range(60):
        a = g.step_resident()
        b = o.step(ref)
        for q, name in enumerate(("clamp_deficit_volume", "source_volume",
                                  "boundary_outflow_volume")):
            va, vb = getattr(a, name), getattr(b, name)
            assert va.hex() == vb.hex(), (k, name, va, vb)
            nonzero[q] += vb != 0.0
    if case == "flood256":  # (the final-update clamp itself practically never fires)
        assert nonzero[1] > 0 and nonzero[2] > 0, nonzero


def test_host_mirror_steps_match_oracle(gpu_cls, oracle_built):
    """Opt-in host mirror (swf_set_host_mirror): steady pinned host steps skip
    every host->device copy, a declared edit (host_changed) re-uploads, and
    the results stay bit-identical to the oracle."""
    import torch
    from paper_1705_00614_b200.types import FlowState
    sc = S.floodplain(256, 50.0)
    st = sc.state.copy()
    pin = lambda a: torch.from_numpy(a.copy()).pin_memory().numpy()
    hs = FlowState(st.nx, st.ny, 0.0, pin(st.H), pin(st.HUx), pin(st.HUy))
    cpu_state = st.copy()
    g = make(gpu_cls, sc)
    g.set_host_mirror(True)
    o = make(oracle_built.OracleStepper, sc)
    ingest = []
    for k in range(10):
        if k == 6:  # an edit, declared
            j, i = np.argwhere(hs.H.reshape(st.ny, st.nx) <= sc.params.eps_dry)[7]
            for a in (hs, cpu_state):
                a.H.reshape(st.ny, st.nx)[j, i] += 0.25
            g.host_changed()
        ia = g.step(hs)
        ib = o.step(cpu_state)
        ingest.append(g.last_ingest_bytes())
        assert ia.tau == ib.tau, k
    assert_state_bitwise(hs, cpu_state, "mirrored host steps")
    full = 3 * 8 * st.nx * st.ny
    assert ingest[0] == full and ingest[6] == full, ingest
    assert all(ingest[k] == 0 for k in (1, 2, 3, 4, 5, 7, 8, 9)), ingest
    # a resident call in between invalidates the mirror: the next host step re-uploads
    g.upload(hs)
    g.step(hs)
    assert g.last_ingest_bytes() == full
    o.step(cpu_state)
    assert_state_bitwise(hs, cpu_state, "mirrored host steps after a re-upload")


def test_speculative_division_redo_path_is_exact(gpu_cls, oracle_built):
    """Momenta in the subnormal range make the kernels' speculative divisions
    reject; those tiles are recomputed by the exact redo launches and the
    result stays bit-identical to the oracle."""
    sc = S.floodplain(128, 50.0)
    st = sc.state.copy()
    wet = np.flatnonzero(st.H > 1e-3)
    rng = np.random.default_rng(3)
    pick = rng.choice(wet, 40, replace=False)
    st.HUx[pick] = 3e-310 * rng.choice([-1.0, 1.0], pick.size)
    st.HUy[pick[::2]] = -1e-312
    g = make(gpu_cls, sc)
    o = make(oracle_built.OracleStepper, sc)
    a, b = st.copy(), st.copy()
    redone = 0
    for _ in range(4):
        ia, ib = g.step(a), o.step(b)
        assert ia.tau == ib.tau
        redone += sum(g.redo_counts())
    assert redone > 0
    assert_state_bitwise(a, b, "speculative redo")


def test_cfl_abort_pinned_write_through_restores_state(gpu_cls, oracle_built):
    """The pinned host step writes updated cells straight into the caller's
    arrays during k_step; on a numerical abort they are restored, so the
    caller's state is untouched, as in the reference."""
    import torch
    from paper_1705_00614_b200 import NumericalError
    from paper_1705_00614_b200.types import FlowState
    sc = _cfl_case()
    pin = lambda a: torch.from_numpy(a.copy()).pin_memory().numpy()
    st = FlowState(sc.state.nx, sc.state.ny, sc.state.t, pin(sc.state.H), pin(sc.state.HUx),
                   pin(sc.state.HUy))
    before = st.copy()
    s = make(gpu_cls, sc)
    with pytest.raises(NumericalError, match="particle displacement"):
        s.step(st, 0.1)
    assert_state_bitwise(st, before, "pinned state changed on abort")


@pytest.mark.parametrize("nx,ny,bs", [(97, 53, 16), (33, 130, 8), (161, 17, 7)])
def test_odd_sizes_vs_oracle(gpu_cls, oracle_built, nx, ny, bs):
    """Partial tiles in both directions, odd row lengths (scalar ingest path),
    block sizes that do and do not divide the 32x16 tile: bitwise vs the
    oracle, through the resident path and through pinned host buffers."""
    import torch
    from paper_1705_00614_b200.types import FlowState
    sc = S.floodplain(192, 50.0, window=(11, 23, nx, ny))
    sc.options.block_size = bs
    st = sc.state.copy()
    g = make(gpu_cls, sc)
    o = make(oracle_built.OracleStepper, sc)
    a = st.copy()
    g.upload(a)
    for _ in range(10):
        g.step_resident()
        o.step(st)
    g.download(a)
    assert_state_bitwise(a, st, f"{nx}x{ny} resident")
    pin = lambda v: torch.from_numpy(v.copy()).pin_memory().numpy()
    hs = FlowState(nx, ny, st.t, pin(st.H), pin(st.HUx), pin(st.HUy))
    for _ in range(5):
        g.step(hs)
        o.step(st)
    assert_state_bitwise(hs, st, f"{nx}x{ny} pinned")


@pytest.mark.parametrize("nx,ny", [(96, 70), (97, 70)])
def test_region_loads_tma_and_per_thread_vs_oracle(gpu_cls, oracle_built, nx, ny):
    """k_step stages its tile regions with TMA tensor copies when the row
    stride allows (even nx; out-of-range cells zero-filled by the copy
    engine) and with per-thread loads otherwise: both bitwise vs the oracle
    on a window whose tiles straddle every domain edge."""
    sc = S.floodplain(192, 50.0, window=(40, 60, nx, ny))
    st = sc.state.copy()
    g = make(gpu_cls, sc)
    assert g.region_loads() == ("tma" if nx % 2 == 0 else "threads")
    o = make(oracle_built.OracleStepper, sc)
    a = st.copy()
    g.upload(a)
    for _ in range(12):
        g.step_resident()
        o.step(st)
    g.download(a)
    assert_state_bitwise(a, st, f"{nx}x{ny} ({g.region_loads()})")


@pytest.mark.parametrize("n,win", [(40960, (0, 20000, 40960, 40)), (8192, (4000, 0, 5, 8192))])
def test_extreme_aspect_ratios_vs_oracle(gpu_cls, oracle_built, n, win):
    """Ragged extremes: a 40960-wide, 40-row band (long rows, one partial tile
    row, 1280 tiles per row) and a 5-wide, 8192-tall column (one partial tile
    column): bitwise vs the oracle."""
    sc = S.floodplain(n, 50.0, window=win)
    st = sc.state.copy()
    g = make(gpu_cls, sc)
    o = make(oracle_built.OracleStepper, sc)
    a = st.copy()
    g.upload(a)
    for _ in range(6):
        ia = g.step_resident()
        ib = o.step(st)
        assert ia.tau == ib.tau
    g.download(a)
    assert_state_bitwise(a, st, f"{sc.terrain.nx}x{sc.terrain.ny}")


@pytest.mark.parametrize("nx,ny", [(1, 1), (1, 9), (9, 1), (2, 2)])
def test_degenerate_grids_vs_oracle(gpu_cls, oracle_built, nx, ny):
    """The smallest grids (a single cell, one row, one column): every cell is
    a domain-edge cell of one partial tile; bitwise vs the oracle."""
    from paper_1705_00614_b200.types import (FlowState, PhysicalParams, StepperOptions, Terrain,
                                             TimestepControl)
    n = nx * ny
    T = Terrain(nx, ny, 2.0, 0.0, 0.0, np.linspace(0.0, 0.3, n))
    P = PhysicalParams(n_manning=0.03, nu=0.5)
    st = FlowState(nx, ny, 0.0, np.linspace(1.0, 0.2, n), np.full(n, 0.1), np.full(n, -0.05))
    g = gpu_cls(T, P, TimestepControl(dt_max=0.05), StepperOptions())
    o = oracle_built.OracleStepper(T, P, TimestepControl(dt_max=0.05), StepperOptions())
    a, b = st.copy(), st.copy()
    for _ in range(20):
        ia, ib = g.step(a), o.step(b)
        assert ia.tau == ib.tau
    assert_state_bitwise(a, b, f"{nx}x{ny}")


@pytest.mark.parametrize("what", ["nan_momentum", "inf_momentum", "nan_two_cells"])
def test_non_finite_state_raises_like_the_reference(gpu_cls, oracle_built, what):
    """Non-finite momenta in wet cells ("nulls" of this domain): the step
    aborts with the reference's non-finite-flux error naming the same cell
    (raise_pending_error, stepper.cpp:568-577), on the fused and the staged
    path, and leaves the state untouched."""
    from paper_1705_00614_b200 import NumericalError
    sc = S.floodplain(96, 50.0)
    st = sc.state.copy()
    wet = np.flatnonzero(st.H > 0.5)
    k = wet[len(wet) // 2]
    if what == "nan_momentum":
        st.HUx[k] = np.nan
    elif what == "inf_momentum":
        st.HUy[k] = np.inf
    else:
        st.HUx[k] = np.nan
        st.HUy[wet[len(wet) // 3]] = np.nan
    o = make(oracle_built.OracleStepper, sc, kind="orc")
    with pytest.raises(NumericalError) as eo:
        o.step(st.copy())
    for mode in (0, 1):
        g = make(gpu_cls, sc, mode=mode)
        a = st.copy()
        before = a.copy()
        with pytest.raises(NumericalError) as eg:
            g.step(a)
        assert str(eg.value) == str(eo.value), (mode, str(eg.value), str(eo.value))
        np.testing.assert_array_equal(a.H, before.H)
        np.testing.assert_array_equal(np.isnan(a.HUx), np.isnan(before.HUx))


def test_wrong_sized_state_arrays_are_a_config_error(gpu_cls):
    """a state array whose length is not nx*ny is rejected before
    any copy or native call (the native entry points read and write nx*ny
    doubles), by step, upload and download alike."""
    from paper_1705_00614_b200 import ConfigError
    sc = S.floodplain(32, 50.0)
    s = make(gpu_cls, sc)
    for f in ("H", "HUx", "HUy"):
        st = sc.state.copy()
        setattr(st, f, getattr(st, f)[:-5].copy())
        for call in (s.step, s.upload, s.download):
            with pytest.raises(ConfigError, match=f"state array {f}"):
                call(st)
