"""GPU parity on seeded random scenarios (tests/fuzz_scenarios.py): every
knob of the step path drawn at random, the CUDA path through the C ABI
against the compiled reference (the C restatement where oracle/_ref is
absent), through the three ways the step is driven -- the drop-in
step(FlowState) on pageable arrays, resident steps, and pinned host buffers
(write-through) -- with states, StepInfo and aborts bitwise / verbatim."""
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


@pytest.mark.parametrize("seed", range(150))
def test_random_scenarios_vs_reference(oracle_built, seed):
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper
    from paper_1705_00614_b200.types import FlowState
    kind = "ref" if oracle_built.available("ref") else "orc"
    sc = random_scenario(seed)
    o = make(oracle_built.OracleStepper, sc, kind=kind)
    g = make(CsphTvdStepper, sc)
    so = sc.state.copy()
    how = seed % 3
    if how == 0:
        sg, drv = sc.state.copy(), g
    elif how == 1:
        sg = sc.state.copy()
        drv = _Resident(g, sg)
    else:
        pin = lambda v: torch.from_numpy(np.array(v, copy=True)).pin_memory().numpy()
        st = sc.state
        sg = FlowState(st.nx, st.ny, st.t, pin(st.H), pin(st.HUx), pin(st.HUy))
        drv = g
    k, msg = run_pair(o, drv, so, sg, 20)
    assert_state_bitwise(sg, so, f"seed {seed} ({['pageable', 'resident', 'pinned'][how]}, "
                                 f"{k} steps{', ' + msg if msg else ''})")
