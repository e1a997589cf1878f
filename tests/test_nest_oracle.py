"""Nesting oracle (oracle/nest.py) against the SPEC.md [MODULE] nesting
examples and invariants.  The reference ships no nesting
code, so these known answers are what pins the oracle; the GPU tests
(test_gpu_nest.py) then compare the device path with this oracle bit for bit."""
import numpy as np
import pytest

from helpers import assert_state_bitwise, make
from oracle import nest as N
from paper_1705_00614_b200 import scenarios as S
from paper_1705_00614_b200.types import (BoundaryConfig, EdgeKind, FlowState, PhysicalParams,
                                         StepperOptions, Terrain, TimestepControl)

EPS = 1e-6


def test_ghost_enumeration_covers_band_once():
    w = N.Window(3, 4, 5, 6, r=4, ghost=2)
    fi, fj = N.ghost_cells(w)
    assert fi.size == w.nxf * w.nyf - (4 * 5) * (4 * 6)
    flat = fi + fj * w.nxf
    assert np.unique(flat).size == flat.size
    inner = (fi >= 2) & (fi < w.nxf - 2) & (fj >= 2) & (fj < w.nyf - 2)
    assert not inner.any()


def _coarse(n=16, h=8.0, H=None, b=None):
    b = np.zeros(n * n) if b is None else b
    return Terrain(n, n, h, 0.0, 0.0, b)


def test_prolong_uniform_depth_flat_bed():
    # SPEC.md:374 globally uniform H over flat bed -> ghost H equals that constant
    n, w = 16, N.Window(4, 5, 6, 5, r=4, ghost=2)
    cH = np.full(n * n, 1.375)
    g = N.prolong(w, cH, np.zeros(n * n), np.zeros(n * n), np.zeros(n * n), n,
                  np.zeros(w.nxf * w.nyf), EPS)
    assert np.all(g[0] == 1.375) and np.all(g[1] == 0.0) and np.all(g[2] == 0.0)


def test_prolong_linear_ramp_is_reproduced():
    # SPEC.md:375 linear eta ramp in x, flat bed -> ghost eta reproduces the ramp
    n, h, r = 16, 8.0, 4
    w = N.Window(4, 5, 6, 5, r=r, ghost=2)
    i = np.tile(np.arange(n), n).astype(float)
    cH = 2.0 + 0.01 * (i + 0.5) * h  # eta at coarse cell centres
    g = N.prolong(w, cH, np.zeros(n * n), np.zeros(n * n), np.zeros(n * n), n,
                  np.zeros(w.nxf * w.nyf), EPS)
    fi, fj = N.ghost_cells(w)
    xf = w.i0 * h + ((fi - w.ghost) + 0.5) * (h / r)  # physical x of the fine centres
    np.testing.assert_allclose(g[0], 2.0 + 0.01 * xf, rtol=1e-14, atol=0)


def test_prolong_lake_at_rest_has_no_velocity_and_stays_at_rest(oracle_built):
    # SPEC.md:376 lake at rest over varying bed -> ghost velocities 0 and the
    # fine stage produces no flow
    # (a fully wet lake: at a shoreline the bilinear eta mixes the dry cells'
    # eta = b, which is not a rest state of the fine grid)
    ns = S.nested_floodplain(64, 50.0, (20, 20, 16, 16), 4, 2)
    level = float(max(ns.coarse.terrain.b.max(), ns.fine.terrain.b.max())) + 1.0
    for sc in (ns.coarse, ns.fine):
        sc.state.H = np.maximum(level - sc.terrain.b, 0.0)
        sc.state.H[sc.state.H <= EPS] = 0.0
        sc.params = PhysicalParams()
        sc.sources, sc.wind = [], type(sc.wind)()
    w = N.Window(*ns.window, r=ns.r, ghost=ns.ghost)
    g = N.prolong(w, ns.coarse.state.H, ns.coarse.state.HUx, ns.coarse.state.HUy,
                  ns.coarse.terrain.b, 64, ns.fine.terrain.b, EPS)
    assert np.all(g[1] == 0.0) and np.all(g[2] == 0.0)
    cs = make(oracle_built.OracleStepper, ns.coarse)
    fs = make(oracle_built.OracleStepper, ns.fine)
    nest = N.OracleNest(w, fs, ns.fine.state, ns.fine.terrain.b, EPS)
    for _ in range(5):
        N.coupled_step(cs, ns.coarse.state, ns.coarse.terrain.b, [nest])
    assert np.abs(ns.fine.state.HUx).max() <= 1e-12
    assert np.abs(ns.fine.state.HUy).max() <= 1e-12
    assert np.abs(ns.coarse.state.HUx).max() <= 1e-12


def test_restrict_uniform_checkerboard_and_mass():
    # SPEC.md:382-384
    w = N.Window(2, 3, 4, 3, r=2, ghost=2)
    n = 12
    coarse = FlowState(n, n, 0.0, np.zeros(n * n), np.zeros(n * n), np.zeros(n * n))
    fine = FlowState(w.nxf, w.nyf, 0.0, np.full(w.nxf * w.nyf, 0.75), np.zeros(w.nxf * w.nyf),
                     np.zeros(w.nxf * w.nyf))
    N.restrict(w, fine, coarse, n)
    win = coarse.H.reshape(n, n)[3:6, 2:6]
    assert np.all(win == 0.75)
    fi = np.arange(w.nxf)[None, :] + np.arange(w.nyf)[:, None]
    fine.H = np.where(fi % 2 == 0, 0.0, 2.0).reshape(-1).astype(float)
    N.restrict(w, fine, coarse, n)
    assert np.all(coarse.H.reshape(n, n)[3:6, 2:6] == 1.0)
    rng = np.random.default_rng(3)
    w4 = N.Window(2, 3, 4, 3, r=4, ghost=2)
    fine = FlowState(w4.nxf, w4.nyf, 0.0, rng.uniform(0, 3, w4.nxf * w4.nyf),
                     np.zeros(w4.nxf * w4.nyf), np.zeros(w4.nxf * w4.nyf))
    N.restrict(w4, fine, coarse, n)
    h, hf = 8.0, 2.0
    inner = fine.H.reshape(w4.nyf, w4.nxf)[2:-2, 2:-2]
    m_f = inner.sum() * hf * hf
    m_c = coarse.H.reshape(n, n)[3:6, 2:6].sum() * h * h
    assert abs(m_f - m_c) <= 1e-12 * m_f


def _pair(oracle_built, ns):
    cs = make(oracle_built.OracleStepper, ns.coarse)
    fs = make(oracle_built.OracleStepper, ns.fine)
    w = N.Window(*ns.window, r=ns.r, ghost=ns.ghost)
    return cs, N.OracleNest(w, fs, ns.fine.state, ns.fine.terrain.b, EPS)


def test_one_way_is_bitwise_the_unnested_run(oracle_built):
    # SPEC.md:397 with feedback disabled, global results are bitwise identical
    ns = S.nested_floodplain(64, 50.0, (20, 20, 16, 16), 4, 2)
    plain = ns.coarse.state.copy()
    ps = make(oracle_built.OracleStepper, ns.coarse)
    cs, nest = _pair(oracle_built, ns)
    nest.w.two_way = False
    for _ in range(8):
        N.coupled_step(cs, ns.coarse.state, ns.coarse.terrain.b, [nest])
        ps.step(plain)
    assert_state_bitwise(ns.coarse.state, plain, "one-way")


def test_dry_window_equals_plain_global_step(oracle_built):
    # SPEC.md:390 dry window -> coupled_step equals plain global step
    ns = S.nested_floodplain(64, 50.0, (20, 20, 16, 16), 4, 2)
    for st in (ns.coarse.state, ns.fine.state):
        st.H[:] = 0.0
    # water far from the window only
    ns.coarse.state.H.reshape(64, 64)[2:8, 2:8] = 1.0
    ns.coarse.sources = []
    ns.fine.sources = []
    plain = ns.coarse.state.copy()
    ps = make(oracle_built.OracleStepper, ns.coarse)
    cs, nest = _pair(oracle_built, ns)
    for _ in range(5):
        N.coupled_step(cs, ns.coarse.state, ns.coarse.terrain.b, [nest])
        ps.step(plain)
    assert_state_bitwise(ns.coarse.state, plain, "dry window")
    assert not ns.fine.state.H.any()


def _degenerate(n=48, win=(12, 14, 20, 18), ghost=3):
    """r = 1: the fine grid is a copy of the window plus a ghost band."""
    sc = S.floodplain(n, 50.0)
    sc.sources = []
    i0, j0, ni, nj = win
    nxf, nyf = ni + 2 * ghost, nj + 2 * ghost
    B = sc.terrain.b.reshape(n, n)
    sl = (slice(j0 - ghost, j0 + nj + ghost), slice(i0 - ghost, i0 + ni + ghost))
    take = lambda a: a.reshape(n, n)[sl].reshape(-1).copy()
    ft = Terrain(nxf, nyf, 50.0, (i0 - ghost) * 50.0, (j0 - ghost) * 50.0, take(B))
    fp = PhysicalParams(n_manning=sc.params.n_manning, n_field=take(sc.params.n_field),
                        nu=sc.params.nu, omega_z=sc.params.omega_z)
    fst = FlowState(nxf, nyf, 0.0, take(sc.state.H), take(sc.state.HUx), take(sc.state.HUy))
    fine = S.Scenario("deg-fine", ft, fp, TimestepControl(),
                      StepperOptions(boundaries=BoundaryConfig(EdgeKind.Open, EdgeKind.Open,
                                                               EdgeKind.Open, EdgeKind.Open)),
                      fst, [], sc.wind)
    return S.NestedScenario(sc, fine, win, 1, ghost)


def test_r1_degenerate_window_matches_global(oracle_built):
    # SPEC.md:391 r=1 degenerate window -> global and fine agree per step
    # (with a 3-cell ghost band, the dependency radius of the step)
    ns = _degenerate()
    plain = ns.coarse.state.copy()
    ps = make(oracle_built.OracleStepper, ns.coarse)
    cs, nest = _pair(oracle_built, ns)
    i0, j0, ni, nj = ns.window
    for _ in range(6):
        info, subs = N.coupled_step(cs, ns.coarse.state, ns.coarse.terrain.b, [nest])
        ps.step(plain)
        assert subs == [1]
        fin = ns.fine.state.H.reshape(nj + 6, ni + 6)[3:-3, 3:-3]
        glob = plain.H.reshape(48, 48)[j0:j0 + nj, i0:i0 + ni]
        np.testing.assert_array_equal(fin, glob)
    assert_state_bitwise(ns.coarse.state, plain, "r=1")


def test_flood_wave_mass_balance(oracle_built):
    # SPEC.md:392 total system mass over coupled steps, on a closed,
    # source-free system where the window sits in the path of the wave
    ns = S.nested_floodplain(64, 50.0, (24, 24, 16, 16), 2, 2)
    for sc in (ns.coarse, ns.fine):
        sc.sources = []
        sc.options.boundaries = BoundaryConfig(EdgeKind.Reflective, EdgeKind.Reflective,
                                               EdgeKind.Reflective, EdgeKind.Reflective)
    ns.fine.options.boundaries = BoundaryConfig(EdgeKind.Open, EdgeKind.Open, EdgeKind.Open,
                                                EdgeKind.Open)
    w = N.Window(*ns.window, r=ns.r, ghost=ns.ghost)
    N.restrict(w, ns.fine.state, ns.coarse.state, 64)  # consistent start
    cs, nest = _pair(oracle_built, ns)
    area = ns.coarse.terrain.h ** 2
    m0 = ns.coarse.state.H.sum() * area
    ledger = 0.0
    for _ in range(100):
        info, _ = N.coupled_step(cs, ns.coarse.state, ns.coarse.terrain.b, [nest])
        ledger += N.coupled_step.clamp + info.clamp_deficit_volume
    m1 = ns.coarse.state.H.sum() * area
    # with the flux correction the coupled system is
    # conservative to round-off up to the logged clamp volumes (wet/dry fronts
    # across the window edge); 1.4e-3 relative drift over these 100 steps
    # without the correction
    assert abs((m1 - m0) - ledger) <= 1e-11 * m0, (m1 - m0, ledger)
    assert abs(ledger) < 1e-3 * m0
