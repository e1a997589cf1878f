"""The C restatement against the compiled reference on seeded random
scenarios (tests/fuzz_scenarios.py): states, StepInfo and aborts bitwise /
verbatim.  Pins the oracle beyond the crafted goldens.  CPU only; skipped
where the reference could not be compiled (oracle/_ref absent)."""
import pytest

from fuzz_scenarios import random_scenario, run_pair
from helpers import assert_state_bitwise, make


@pytest.mark.parametrize("seed", range(150))
def test_restatement_equals_reference_on_random_scenarios(oracle_built, seed):
    if not oracle_built.available("ref"):
        pytest.skip("the compiled reference (oracle/_ref) is not present")
    sc = random_scenario(seed)
    a = make(oracle_built.OracleStepper, sc, kind="orc")
    b = make(oracle_built.OracleStepper, sc, kind="ref")
    sa, sb = sc.state.copy(), sc.state.copy()
    run_pair(a, b, sa, sb, 20)
    assert_state_bitwise(sa, sb, f"seed {seed}")
