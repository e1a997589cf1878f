"""Configuration fuzzing: seeded random scenarios (tests/fuzz_scenarios.py)
with one field made invalid or extreme -- Courant number, dt bounds, cell
size, a bed / Manning / state value (NaN, inf, negative), block size, wind
or hydrograph times out of order, source rectangles outside the grid or
inverted -- run through the compiled reference and the CUDA drop-in: both
must reject with the same exception type and message at the same call, or
both accept and step to bitwise-equal states (NaN cells, where a non-finite
parameter the reference accepts produces them, in the same places)."""
import copy
import os

import numpy as np
import pytest

from fuzz_scenarios import random_scenario
from helpers import make
from paper_1705_00614_b200.types import CellRect, HydrographSample, WindSample

pytestmark = pytest.mark.gpu


def _mutate(sc, rng):
    sc = copy.deepcopy(sc)
    n = sc.terrain.nx * sc.terrain.ny
    k = int(rng.integers(0, n))
    bad = float(rng.choice([np.nan, np.inf, -np.inf, -1.0, 0.0, -0.0, 1e300, -1e-300]))
    what = int(rng.integers(0, 14))
    if what == 0:
        sc.control.courant = float(rng.choice([0.0, 1.0, 1.5, -0.2, np.nan]))
    elif what == 1:
        sc.control.dt_max = float(rng.choice([0.0, -1.0, np.nan, 1e-12]))
    elif what == 2:
        sc.control.dt_min = float(rng.choice([0.0, -1e-9, sc.control.dt_max, 2 * sc.control.dt_max]))
    elif what == 3:
        sc.terrain.h = float(rng.choice([0.0, -1.0, np.nan, np.inf]))
    elif what == 4:
        sc.terrain.b = sc.terrain.b.copy()
        sc.terrain.b[k] = bad
    elif what == 5:
        sc.params.n_manning = float(rng.choice([-0.01, np.nan, np.inf, 0.0]))
        sc.params.n_field = None
    elif what == 6:
        sc.params.n_field = np.full(n, 0.03)
        sc.params.n_field[k] = bad
    elif what == 7:
        sc.options.block_size = int(rng.choice([0, -1, -16]))
    elif what == 8:
        sc.state.H = sc.state.H.copy()
        sc.state.H[k] = bad
    elif what == 9:
        sc.state.HUx = sc.state.HUx.copy()
        sc.state.HUx[k] = bad
    elif what == 10:  # wind times not increasing, or a NaN component
        s = [WindSample(0.0, 3.0, 1.0), WindSample(5.0, -2.0, 4.0)]
        if rng.random() < 0.5:
            s[1].t = float(rng.choice([0.0, -1.0]))
        else:
            s[1].wx = np.nan
        sc.wind.series = s
    elif what in (11, 12, 13) and sc.sources:
        s = sc.sources[int(rng.integers(0, len(sc.sources)))]
        if what == 11:  # rectangle outside the grid or inverted
            c = s.cells
            s.cells = CellRect(*[(c.i0, c.j0, sc.terrain.nx, c.j1), (c.i1 + 1, c.j0, c.i1, c.j1),
                                 (-1, c.j0, c.i1, c.j1), (c.i0, c.j0, c.i1, sc.terrain.ny + 3)]
                               [int(rng.integers(0, 4))])
        elif what == 12:  # hydrograph times not increasing / empty / NaN rate
            s.hydrograph = [HydrographSample(1.0, 5.0), HydrographSample(1.0, 6.0)] \
                if rng.random() < 0.5 else []
        else:
            s.rate = float(rng.choice([np.nan, -1e-3, np.inf]))
            s.source_velocity.x = float(rng.choice([np.nan, 0.5]))
    else:
        sc.terrain.h = float(rng.choice([1e-300, 1e300]))
    return sc, what


def _outcome(cls, sc, **kw):
    """('ok', state) or (exception type name, message, call)."""
    call = "create"
    try:
        s = cls(sc.terrain, sc.params, sc.control, sc.options, **kw)
        call = "set_wind"
        if sc.wind.any():
            s.set_wind(sc.wind)
        call = "set_sources"
        if sc.sources:
            s.set_sources(sc.sources)
        st = sc.state.copy()
        for q in range(3):
            call = f"step {q}"
            s.step(st)
        return ("ok", st)
    except Exception as e:  # noqa: BLE001 -- compared between the two
        return (type(e).__name__, str(e), call)


# SWF_FUZZ_SEEDS widens the sweep (profiles/fuzz_config_r3zz.txt ran 2000)
@pytest.mark.parametrize("seed", range(int(os.environ.get("SWF_FUZZ_SEEDS", "120"))))
def test_invalid_and_extreme_configs_like_the_reference(oracle_built, seed):
    from paper_1705_00614_b200 import CsphTvdStepper
    kind = "ref" if oracle_built.available("ref") else "orc"
    rng = np.random.default_rng(77_000 + seed)
    sc, what = _mutate(random_scenario(seed), rng)
    ro = _outcome(oracle_built.OracleStepper, sc, kind=kind)
    go = _outcome(CsphTvdStepper, sc)
    if ro[0] == "ok" or go[0] == "ok":
        assert ro[0] == go[0] == "ok", (what, ro, go)
        # non-finite parameters the reference accepts (a NaN wind component,
        # a NaN or infinite Manning n) give NaN states: the NaN cells must be
        # the same ones; their payload and sign bits are the hardware's
        # default NaN (x86: 0xfff8..., the GPU: 0x7fff...), which IEEE 754
        # leaves unspecified, so only the other cells compare bit for bit
        for f in ("H", "HUx", "HUy"):
            a, b = getattr(go[1], f), getattr(ro[1], f)
            na, nb = np.isnan(a), np.isnan(b)
            assert np.array_equal(na, nb), (what, f, int(na.sum()), int(nb.sum()))
            assert np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64)), (what, f)
        assert go[1].t == ro[1].t
    else:
        assert go == ro, (what, ro, go)


def test_abort_cell_from_a_redone_tile_wins_in_block_order(oracle_built):
    """Seed 7974 (a NaN rain rate): at step 1 two tiles hit the h/2
    displacement abort; the one earlier in the reference's block order had a
    rejected speculative division and is recomputed by the exact redo launch
    after the other had published its error.  The abort must still name the
    first cell in block order (it named the later one while an error raised
    by the same step stopped the redo; StepScalars::step_open)."""
    test_invalid_and_extreme_configs_like_the_reference(oracle_built, 7974)
