"""GPU parity on seeded random scenarios (tests/fuzz_scenarios.py): every
knob of the step path drawn at random, the CUDA path through the C ABI
against the compiled reference (the C restatement where oracle/_ref is
absent), through every way the step is driven -- the drop-in
step(FlowState) on pageable arrays, resident steps, pinned host buffers
(write-through), pinned buffers under the opt-in host mirror, a 20-step
CUDA-graph run (an abort commits the steps before it), and the staged path
(one kernel per reference stage) -- with states,
StepInfo and aborts bitwise / verbatim."""
import os

import numpy as np
import pytest

from fuzz_scenarios import random_scenario, run_pair
from helpers import assert_state_bitwise, make

pytestmark = pytest.mark.gpu


class _Resident:
    """step(state) over the device-resident path: upload once, swf_step,
    download after every step (so the comparison sees each state)."""

    def __init__(self, g, st):
        self.g = g
        g.upload(st)

    def step(self, st, dt_cap=0.0):
        info = self.g.step_resident(dt_cap)
        self.g.download(st)
        return info


DRIVERS = ("pageable", "resident", "pinned", "pinned+mirror", "run", "staged")


# SWF_FUZZ_SEEDS widens the sweep (profiles/fuzz_drivers_r3zz.txt ran 3000)
@pytest.mark.parametrize("seed", range(int(os.environ.get("SWF_FUZZ_SEEDS", "150"))))
def test_random_scenarios_vs_reference(oracle_built, seed):
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper
    from paper_1705_00614_b200.types import FlowState
    kind = "ref" if oracle_built.available("ref") else "orc"
    sc = random_scenario(seed)
    o = make(oracle_built.OracleStepper, sc, kind=kind)
    how = DRIVERS[seed % len(DRIVERS)]
    # "staged": the one-kernel-per-reference-stage path (swf_stage.cu)
    g = make(CsphTvdStepper, sc, mode=1) if how == "staged" else make(CsphTvdStepper, sc)
    so = sc.state.copy()
    # a third of the seeds cap the step (stepper.hpp:84-86: tau = min(CFL tau, dt_cap))
    # (every driver meets capped and uncapped seeds: the cap cycles per driver round)
    dt_cap = [0.0, 0.0, float(np.random.default_rng(seed).uniform(1e-4, 0.5))][
        (seed // len(DRIVERS)) % 3]
    if how == "run":  # 20 steps in one CUDA-graph batch; an abort commits the steps before it
        from paper_1705_00614_b200 import NumericalError
        sg = sc.state.copy()
        g.upload(sg)
        k, msg = 20, None
        for q in range(20):
            try:
                last = o.step(so, dt_cap)
            except NumericalError as e:
                k, msg = q, str(e)
                break
        if msg is None:
            done, info = g.run(20, dt_cap)
            assert done == 20
            for f in ("tau", "clamp_deficit_volume", "source_volume", "boundary_outflow_volume"):
                assert getattr(info, f) == getattr(last, f), f
        else:
            with pytest.raises(NumericalError) as eg:
                g.run(20, dt_cap)
            assert str(eg.value) == msg
        g.download(sg)
    else:
        if how in ("pageable", "resident", "staged"):
            sg = sc.state.copy()
        else:
            pin = lambda v: torch.from_numpy(np.array(v, copy=True)).pin_memory().numpy()
            st = sc.state
            sg = FlowState(st.nx, st.ny, st.t, pin(st.H), pin(st.HUx), pin(st.HUy))
            if how == "pinned+mirror":
                g.set_host_mirror(True)
        drv = _Resident(g, sg) if how == "resident" else g
        k, msg = run_pair(o, drv, so, sg, 20, dt_cap)
    assert_state_bitwise(sg, so, f"seed {seed} ({how}, cap {dt_cap}, {k} steps{', ' + msg if msg else ''})")


@pytest.mark.parametrize("seed", range(60))
def test_random_scenarios_row_strips_vs_single_grid(seed):
    """The same random scenarios split into 2-4 row strips (virtual ranks on
    this GPU; synchronous or asynchronous protocol): the assembled owned rows
    bitwise equal to the single grid (itself bitwise to the reference above)."""
    from paper_1705_00614_b200 import CsphTvdStepper, NumericalError
    from paper_1705_00614_b200 import multigpu as M
    from fuzz_scenarios import window
    from helpers import assert_bitwise
    sc = random_scenario(seed)
    ny, nx, bs = sc.terrain.ny, sc.terrain.nx, sc.options.block_size
    parts = 2 + seed % 3
    try:
        bounds = M.strip_bounds(ny, parts, bs)
    except ValueError:
        pytest.skip("grid too small for that many strips of >= 3 rows")
    one = make(CsphTvdStepper, sc)
    st = sc.state.copy()
    one.upload(st)
    try:
        done, _ = one.run(15)
    except NumericalError:
        pytest.skip("the scenario aborts (covered against the reference above)")
    one.download(st)
    strips = []
    for j0, j1 in bounds:
        w0, w1 = M.window_rows(j0, j1, ny)
        ws = window(sc, w0, w1)
        s = M.Strip(ws, ny, j0, j1, ws.global_sources, ws.wind)
        s.upload(ws.state.H, ws.state.HUx, ws.state.HUy, 0.0)
        strips.append((s, ws, w0))
    if seed % 2:  # (block sizes not dividing 16: no interior/ghost overlap, same results)
        res = M.local_steps_async([s for s, _, _ in strips], 15)
        assert all(d == 15 for d, _ in res)
    else:
        for _ in range(15):
            M.local_step([s for s, _, _ in strips])
    out = {f: np.empty(nx * ny) for f in ("H", "HUx", "HUy")}
    for (s, ws, w0), (j0, j1) in zip(strips, bounds):
        a = {f: np.empty(ws.terrain.nx * ws.terrain.ny) for f in out}
        assert s.download(a["H"], a["HUx"], a["HUy"]) == st.t
        r0 = (j0 - w0) * nx
        for f in out:
            out[f][j0 * nx:j1 * nx] = a[f][r0:r0 + (j1 - j0) * nx]
    for f in out:
        assert_bitwise(out[f], getattr(st, f), f"seed {seed} {parts} strips {f}")


STAGE_SCRATCH = ["fn_fx", "fn_fy", "fn_fric_x", "fn_fric_y", "fn_sigma", "fm_fx", "fm_fy",
                 "fm_fric_x", "fm_fric_y", "fm_sigma", "Ht", "HVtx", "HVty", "drx", "dry", "Fh",
                 "Fvx", "Fvy", "sigma", "src_vx", "src_vy"]


@pytest.mark.parametrize("seed", range(40))
def test_random_scenarios_stagewise_vs_reference(oracle_built, seed):
    """The eight stage methods (stepper.hpp:88-96) one by one on the random
    scenarios, every scratch accessor (stepper.hpp:102-119) and the block
    mask bitwise against the compiled reference after each stage sequence;
    aborts inside a stage with the reference's type and message."""
    from paper_1705_00614_b200 import CsphTvdStepper
    from helpers import assert_bitwise
    kind = "ref" if oracle_built.available("ref") else "orc"
    sc = random_scenario(seed)
    a = make(oracle_built.OracleStepper, sc, kind=kind)
    b = make(CsphTvdStepper, sc)
    sa, sb = sc.state.copy(), sc.state.copy()

    def both(fa, fb):
        ea = eb = ra = rb = None
        try:
            ra = fa()
        except Exception as e:  # noqa: BLE001 -- compared below
            ea = e
        try:
            rb = fb()
        except Exception as e:  # noqa: BLE001
            eb = e
        assert (type(ea).__name__, str(ea)) == (type(eb).__name__, str(eb))
        return ea is not None, ra, rb

    for step in range(4):
        for name in ("begin_step", "compute_forces"):
            stop, _, _ = both(lambda: getattr(a, name)(sa), lambda: getattr(b, name)(sb))
            if stop:
                return
        stop, ta, tb = both(lambda: a.compute_dt(sa), lambda: b.compute_dt(sb))
        if stop:
            return
        assert ta == tb
        for name in ("predictor", "mid_forces", "corrector", "flux"):
            stop, _, _ = both(lambda: getattr(a, name)(sa, ta), lambda: getattr(b, name)(sb, tb))
            if stop:
                return
        for nm in STAGE_SCRATCH:
            assert_bitwise(b.scratch(nm), a.scratch(nm), f"seed {seed} step {step} {nm}")
        ma, mb = a.mask(), b.mask()
        assert np.array_equal(ma.interior_wet, mb.interior_wet)
        assert np.array_equal(ma.halo_wet, mb.halo_wet)
        both(lambda: a.final_update(sa, ta), lambda: b.final_update(sb, tb))
        assert_state_bitwise(sb, sa, f"seed {seed} step {step}")
        assert b._volumes() == a._volumes()


@pytest.mark.parametrize("seed", range(40))
def test_random_scenarios_strip_host_steps(seed):
    """The strips' host-buffer step (swf_strip_host_phase1/2, the multi-GPU
    e2e path) on the random scenarios: every strip reads its window from one
    pinned global state and writes its owned cells back in place, bitwise
    equal to the single grid."""
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper, NumericalError
    from paper_1705_00614_b200 import multigpu as M
    from fuzz_scenarios import window
    from helpers import assert_bitwise
    sc = random_scenario(seed)
    nx, ny, bs = sc.terrain.nx, sc.terrain.ny, sc.options.block_size
    try:
        bounds = M.strip_bounds(ny, 2 + seed % 2, bs)
    except ValueError:
        pytest.skip("grid too small for that many strips of >= 3 rows")
    one = make(CsphTvdStepper, sc)
    ref = sc.state.copy()
    one.upload(ref)
    try:
        one.run(10)
    except NumericalError:
        pytest.skip("the scenario aborts (covered against the reference above)")
    one.download(ref)
    pin = lambda a: torch.from_numpy(np.array(a, copy=True)).pin_memory().numpy()
    H, X, Y = pin(sc.state.H), pin(sc.state.HUx), pin(sc.state.HUy)
    strips = []
    for j0, j1 in bounds:
        w0, w1 = M.window_rows(j0, j1, ny)
        ws = window(sc, w0, w1)
        strips.append((M.Strip(ws, ny, j0, j1, ws.global_sources, ws.wind), w0 * nx))
    t = 0.0
    for _ in range(10):
        sp = [s.host_phase1(H[o:], X[o:], Y[o:], t) for s, o in strips]
        g = max(sp)
        ts = [s.host_phase2(H[o:], X[o:], Y[o:], g)[0] for s, o in strips]
        assert len(set(ts)) == 1
        t = ts[0]
    assert t == ref.t
    assert_bitwise(H, ref.H, f"seed {seed} H")
    assert_bitwise(X, ref.HUx, f"seed {seed} HUx")
    assert_bitwise(Y, ref.HUy, f"seed {seed} HUy")
