"""Runs scenarios on the opt-in FAST build (libswflood_cuda_fast.so) in a
process of its own (the library is loaded once per process) and saves the
states: test infrastructure for tests/test_gpu_fast.py.

    SWF_FLAVOR=fast python tests/fast_runner.py OUT.npz CASE STEPS DT_CAP
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def cases():
    from paper_1705_00614_b200 import scenarios as S
    return {
        "c1_dry_n002": lambda: S.dam_break_1d(False, 0.02),
        "c1_wet_n0": lambda: S.dam_break_1d(True, 0.0),
        "c2_256": lambda: S.circular_dam_break(256, 8.0, 32, n_manning=0.03),
        "c3_crop": lambda: S.floodplain(16384, 50.0, window=(6144, 14336, 256, 256)),  # 30 % wet
        "c3_rain": lambda: S.floodplain(16384, 50.0, window=(1980, 10180, 256, 256)),  # rain edge
        "lake128": lambda: S.lake_at_rest(128),
    }


def main():
    out, case, steps, dt_cap = sys.argv[1], sys.argv[2], int(sys.argv[3]), float(sys.argv[4])
    from helpers import make
    from paper_1705_00614_b200 import CsphTvdStepper
    from paper_1705_00614_b200._lib import lib
    sc = cases()[case]()
    s = make(CsphTvdStepper, sc)
    st = sc.state.copy()
    s.upload(st)
    taus = []
    for _ in range(steps):
        taus.append(s.step_resident(dt_cap).tau)
    s.download(st)
    np.savez(out, H=st.H, HUx=st.HUx, HUy=st.HUy, t=st.t, taus=np.array(taus),
             flavor=lib().swf_build_flavor().decode())


if __name__ == "__main__":
    main()
