"""The pybind11 module `swflood_native` (host/swflood_pybind.cpp): the
reference's C++ API (grid.hpp, sources.hpp, stepper.hpp) from Python, over
the C++ drop-in and the CUDA library.  CPU: types, numpy views, error
mapping, no CPU fallback.  GPU: steps bit-identical to the oracle."""
import numpy as np
import pytest

from conftest import has_gpu
from helpers import assert_state_bitwise, make
from paper_1705_00614_b200 import scenarios as S

sw = pytest.importorskip("paper_1705_00614_b200.swflood_native")


def to_native(sc):
    """A scenario (paper_1705_00614_b200.types) as swflood_native objects."""
    T = sw.Terrain(sc.terrain.nx, sc.terrain.ny, sc.terrain.h, sc.terrain.x0, sc.terrain.y0,
                   sc.terrain.b)
    P = sw.PhysicalParams()
    for f in ("g", "n_manning", "nu", "omega_z", "c_a", "rho_air", "rho_water", "eps_dry"):
        setattr(P, f, getattr(sc.params, f))
    if sc.params.n_field is not None:
        P.n_field = sc.params.n_field
    K = sw.TimestepControl(sc.control.courant, sc.control.dt_max, sc.control.dt_min)
    O = sw.StepperOptions()
    O.block_size = sc.options.block_size
    O.skip_dry_blocks = sc.options.skip_dry_blocks
    bc = sw.BoundaryConfig()
    for e in ("west", "east", "south", "north"):
        setattr(bc, e, sw.EdgeKind(int(getattr(sc.options.boundaries, e))))
    O.boundaries = bc
    W = sw.WindForcing([sw.WindSample(s.t, s.wx, s.wy) for s in sc.wind.series])
    srcs = []
    for s in sc.sources:
        n = sw.SourceSpec()
        n.kind = sw.SourceSpec.Kind(int(s.kind))
        n.name = s.name
        n.cells = sw.CellRect(s.cells.i0, s.cells.j0, s.cells.i1, s.cells.j1)
        n.hydrograph = [sw.HydrographSample(h.t, h.q) for h in s.hydrograph]
        n.rate = s.rate
        n.source_velocity = sw.Vec2(s.source_velocity.x, s.source_velocity.y)
        srcs.append(n)
    st = sw.FlowState.dry(T)
    st.H[:], st.HUx[:], st.HUy[:] = sc.state.H, sc.state.HUx, sc.state.HUy
    st.t = sc.state.t
    return T, P, K, O, W, srcs, st


def test_types_and_views():
    sc = S.floodplain(64, 50.0)
    T, P, K, O, W, srcs, st = to_native(sc)
    assert T.cells() == 64 * 64 and T.idx(3, 2) == 2 * 64 + 3
    np.testing.assert_array_equal(T.b, sc.terrain.b)
    v = st.H
    v[0] = 7.0  # a view onto the C++ vector, not a copy
    assert st.H[0] == 7.0
    assert len(W.series) == len(sc.wind.series) and len(srcs) == len(sc.sources)
    assert srcs[0].discharge_at(0.0) == sc.sources[0].discharge_at(0.0)


def test_config_errors_and_no_cpu_fallback():
    T = sw.Terrain(4, 4, 1.0, 0.0, 0.0, np.zeros(16))
    with pytest.raises(sw.ConfigError, match="Courant"):
        sw.CsphTvdStepper(T, sw.PhysicalParams(), sw.TimestepControl(courant=1.5))
    bad = sw.Terrain(4, 4, 1.0, 0.0, 0.0, np.zeros(15))
    with pytest.raises(sw.ConfigError, match="bed array size mismatch"):
        sw.CsphTvdStepper(bad, sw.PhysicalParams(), sw.TimestepControl())
    if not has_gpu():
        with pytest.raises(RuntimeError, match="CUDA|device"):
            sw.CsphTvdStepper(T, sw.PhysicalParams(), sw.TimestepControl())


@pytest.mark.gpu
def test_native_steps_match_oracle(oracle_built):
    sc = S.floodplain(96, 50.0)
    T, P, K, O, W, srcs, st = to_native(sc)
    g = sw.CsphTvdStepper(T, P, K, O)
    g.set_wind(W)
    g.set_sources(srcs)
    o = make(oracle_built.OracleStepper, sc)
    ref = sc.state.copy()
    for _ in range(10):
        a = g.step(st)
        b = o.step(ref)
        assert a.tau == b.tau
        assert (a.lagrangian_blocks, a.flux_blocks) == (b.lagrangian_blocks, b.flux_blocks)
    out = sc.state.copy()
    out.H[:], out.HUx[:], out.HUy[:], out.t = st.H, st.HUx, st.HUy, st.t
    assert_state_bitwise(out, ref, "pybind steps")


@pytest.mark.gpu
def test_native_numerical_error_leaves_state():
    T = sw.Terrain(64, 8, 1.0, 0.0, 0.0, np.zeros(64 * 8))
    st = sw.FlowState.dry(T)
    st.H[:] = 1.0
    st.HUx[:] = 50.0  # CFL tau ~ 0.5 * 1 / 53 m/s falls below dt_min = 0.05
    g = sw.CsphTvdStepper(T, sw.PhysicalParams(), sw.TimestepControl(0.5, 10.0, 0.05))
    before = st.H.copy(), st.HUx.copy()
    with pytest.raises(sw.NumericalError, match="abort floor"):
        g.step(st)
    np.testing.assert_array_equal(st.H, before[0])
    np.testing.assert_array_equal(st.HUx, before[1])


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [2, 3])
def test_native_multi_device_group_matches_oracle(oracle_built, devices):
    """StepperOptions.devices > 1: the stepper drives one row strip per device
    from this process (swf_group_*: peer-linked strips, event-ordered streams,
    device-side speed max).  With one GPU the strips share it -- the same code
    path; results stay bit-identical to the single-grid oracle."""
    sc = S.floodplain(128, 50.0)
    T, P, K, O, W, srcs, st = to_native(sc)
    O.devices = devices
    g = sw.CsphTvdStepper(T, P, K, O)
    g.set_wind(W)
    g.set_sources(srcs)
    o = make(oracle_built.OracleStepper, sc)
    ref = sc.state.copy()
    for _ in range(8):
        a = g.step(st)
        b = o.step(ref)
        assert a.tau == b.tau
        assert (a.lagrangian_blocks, a.flux_blocks, a.total_blocks) == \
            (b.lagrangian_blocks, b.flux_blocks, b.total_blocks)
        assert a.active_fraction == b.active_fraction
    out = sc.state.copy()
    out.H[:], out.HUx[:], out.HUy[:], out.t = st.H, st.HUx, st.HUy, st.t
    assert_state_bitwise(out, ref, f"{devices}-device group")
    with pytest.raises(sw.ConfigError, match="devices == 1"):
        g.begin_step(st)


@pytest.mark.gpu
def test_native_multi_device_abort_leaves_state():
    T = sw.Terrain(64, 64, 1.0, 0.0, 0.0, np.zeros(64 * 64))
    st = sw.FlowState.dry(T)
    st.H[:] = 1.0
    st.HUx[:] = 50.0
    O = sw.StepperOptions()
    O.devices = 2
    g = sw.CsphTvdStepper(T, sw.PhysicalParams(), sw.TimestepControl(0.5, 10.0, 0.05), O)
    before = st.H.copy(), st.HUx.copy(), st.t
    with pytest.raises(sw.NumericalError, match="abort floor"):
        g.step(st)
    np.testing.assert_array_equal(st.H, before[0])
    np.testing.assert_array_equal(st.HUx, before[1])
    assert st.t == before[2]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(60))
def test_native_group_random_scenarios_vs_reference(oracle_built, seed):
    """The C++ drop-in with StepperOptions.devices = 2 or 3 (the in-process
    swf_group; strips share this GPU) on the seeded random scenarios of
    tests/fuzz_scenarios.py, step by step against the compiled reference:
    state, tau, block counts and aborts (same step, same message)."""
    from fuzz_scenarios import random_scenario
    sc = random_scenario(seed)
    T, P, K, O, W, srcs, st = to_native(sc)
    O.devices = 2 + seed % 2
    try:
        g = sw.CsphTvdStepper(T, P, K, O)
    except sw.ConfigError as e:
        assert "too many devices" in str(e) or "block rows" in str(e), str(e)
        pytest.skip(str(e))
    if sc.wind.any():
        g.set_wind(W)
    if srcs:
        g.set_sources(srcs)
    kind = "ref" if oracle_built.available("ref") else "orc"
    o = make(oracle_built.OracleStepper, sc, kind=kind)
    ref = sc.state.copy()
    for k in range(15):
        ea = eb = None
        try:
            a = g.step(st)
        except (sw.NumericalError, sw.ConfigError) as e:
            ea = e
        try:
            b = o.step(ref)
        except Exception as e:  # noqa: BLE001 -- compared below
            eb = e
        if ea or eb:
            assert ea is not None and eb is not None, (k, ea, eb)
            assert str(ea) == str(eb), (k, str(ea), str(eb))
            break
        assert a.tau == b.tau, k
        assert (a.lagrangian_blocks, a.flux_blocks, a.total_blocks) == \
            (b.lagrangian_blocks, b.flux_blocks, b.total_blocks), k
    out = sc.state.copy()
    out.H[:], out.HUx[:], out.HUy[:], out.t = st.H, st.HUx, st.HUy, st.t
    assert_state_bitwise(out, ref, f"seed {seed}, {O.devices}-device group")
