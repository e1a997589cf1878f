"""Exploratory parity sweep (developer tool): the CUDA path against the
compiled reference on many seeded random scenarios (tests/fuzz_scenarios.py).
    python tools/fuzz_sweep.py FIRST COUNT [STEPS]
Prints one JSON line per failing seed and a summary line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from fuzz_scenarios import random_scenario, run_pair  # noqa: E402
from helpers import assert_state_bitwise, make  # noqa: E402


def main():
    import torch
    from oracle import pyorc
    from paper_1705_00614_b200 import CsphTvdStepper
    from paper_1705_00614_b200.types import FlowState
    first, count = int(sys.argv[1]), int(sys.argv[2])
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    kind = "ref" if pyorc.available("ref") else "orc"
    t0 = time.time()
    bad = aborts = 0
    for seed in range(first, first + count):
        sc = random_scenario(seed)
        how = seed % 3
        try:
            o = make(pyorc.OracleStepper, sc, kind=kind)
            g = make(CsphTvdStepper, sc)
            so = sc.state.copy()
            if how == 2:
                pin = lambda v: torch.from_numpy(np.array(v, copy=True)).pin_memory().numpy()
                st = sc.state
                sg = FlowState(st.nx, st.ny, st.t, pin(st.H), pin(st.HUx), pin(st.HUy))
            else:
                sg = sc.state.copy()
            if how == 1:
                class R:
                    def __init__(s):
                        g.upload(sg)

                    def step(s, st, cap=0.0):
                        i = g.step_resident(cap)
                        g.download(st)
                        return i
                drv = R()
            else:
                drv = g
            k, msg = run_pair(o, drv, so, sg, steps)
            aborts += msg is not None
            assert_state_bitwise(sg, so, f"seed {seed}")
        except AssertionError as e:
            bad += 1
            print(json.dumps({"seed": seed, "how": how, "error": str(e)[:400]}), flush=True)
    print(json.dumps({"kind": kind, "seeds": count, "first": first, "steps": steps, "failed": bad,
                      "aborted_runs": aborts, "seconds": round(time.time() - t0, 1)}))


if __name__ == "__main__":
    main()
