"""Debug the FAST build: step a case with a NaN check after every step."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import fast_runner
from helpers import make
from paper_1705_00614_b200 import CsphTvdStepper
case, steps, dt = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
sc = fast_runner.cases()[case]()
s = make(CsphTvdStepper, sc)
st = sc.state.copy()
s.upload(st)
for k in range(steps):
    info = s.step_resident(dt)
    s.download(st)
    bad = ~np.isfinite(st.H) | ~np.isfinite(st.HUx) | ~np.isfinite(st.HUy)
    if bad.any() or not np.isfinite(info.tau):
        idx = np.flatnonzero(bad)[:5]
        print("step", k, "tau", info.tau, "bad", int(bad.sum()), [(int(i) % st.nx, int(i) // st.nx) for i in idx])
        break
else:
    print("no NaN in", steps, "steps; tau", info.tau)
print("lib", os.environ.get("SWF_LIB"), os.environ.get("SWF_FLAVOR"))
