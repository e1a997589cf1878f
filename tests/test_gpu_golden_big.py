"""Parity at the sizes BASELINE.json states: C2 at its full
2048^2 over 1000 steps, the wettest 2048^2 diagonal crop of C3 and a 1024^2
crop of C5 (h = 25 m, all physics and the rain source) over 200 steps --
bit for bit against digests of the REAL reference's trajectories
(tests/golden/golden_big.json, generated from oracle/_ref by
tests/golden/make_golden.py --big), every step's tau included."""
import json
import os

import numpy as np
import pytest

from helpers import digest, make
from paper_1705_00614_b200 import scenarios as S

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "golden_big.json")) as f:
    GB = json.load(f)["cases"]

FACTORIES = {
    "c2_2048_full": lambda: S.circular_dam_break(2048, 8.0, 256, n_manning=0.03),
    "c3_crop2048_k5": lambda: S.build("C3", window=(10240, 10240, 2048, 2048)),
    "c5_crop1024_rain": lambda: S.build("C5", window=(3584, 19968, 1024, 1024)),
}


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("name", sorted(FACTORIES))
def test_config_size_trajectory(name, mode):
    from paper_1705_00614_b200 import CsphTvdStepper
    case = GB[name]
    sc = FACTORIES[name]()
    assert sc.cells() == case["cells"]
    s = make(CsphTvdStepper, sc, mode=mode)
    st = sc.state.copy()
    s.upload(st)
    taus = []
    info = None
    for _ in range(case["steps"]):
        info = s.step_resident(case["dt_cap"])
        taus.append(info.tau.hex())
    s.download(st)
    bad = [k for k, (a, b) in enumerate(zip(taus, case["taus"])) if a != b]
    assert not bad, f"tau differs from step {bad[0]}: {taus[bad[0]]} vs {case['taus'][bad[0]]}"
    assert st.t.hex() == case["t"]
    assert digest(st) == case["sha256"]
    li = case["last_info"]
    assert (info.lagrangian_blocks, info.flux_blocks, info.total_blocks) == \
        (li["lagrangian_blocks"], li["flux_blocks"], li["total_blocks"])
    assert info.active_fraction.hex() == li["active_fraction"]
    for k in ("clamp_deficit_volume", "source_volume", "boundary_outflow_volume"):
        assert getattr(info, k).hex() == li[k], k  # the reference's summation order
    assert int((st.H > sc.params.eps_dry).sum()) == case["wet_cells_end"]
    s.close()


def test_config_size_host_buffer_steps():
    """The drop-in host-buffer step(FlowState&) on pinned arrays over the
    C5 crop's whole trajectory (sparse ingest + write-through every step)."""
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper
    from paper_1705_00614_b200.types import FlowState
    name = "c5_crop1024_rain"
    case = GB[name]
    sc = FACTORIES[name]()
    pin = lambda a: torch.from_numpy(np.array(a, copy=True)).pin_memory().numpy()
    st = FlowState(sc.state.nx, sc.state.ny, 0.0, pin(sc.state.H), pin(sc.state.HUx),
                   pin(sc.state.HUy))
    s = make(CsphTvdStepper, sc)
    for k in range(case["steps"]):
        assert s.step(st).tau.hex() == case["taus"][k]
    assert st.t.hex() == case["t"]
    assert digest(st) == case["sha256"]
    s.close()
