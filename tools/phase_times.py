"""k_step phase breakdown from a -DSWF_PHASE_TIMING build (developer tool).
    SWF_LIB=paper_1705_00614_b200/variants/libswf_phase.so python tools/phase_times.py C3 5"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper, scenarios as S
    from paper_1705_00614_b200._lib import lib
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    sc = S.build(cfg, device="cuda")
    st = CsphTvdStepper(sc.terrain, sc.params, sc.control, sc.options)
    st.set_wind(sc.wind)
    st.set_sources(sc.sources)
    st.upload(sc.state)
    st.run(3)
    out = (C.c_ulonglong * 16)()
    f = lib().swf_debug_phase_cycles
    f(out, 1)
    st.run(K)
    f(out, 1)
    names = ["1a loads", "1b predictor", "2 forces+corrector", "3x slopes", "4x faces",
             "3y slopes", "4y faces", "5 final"]
    tot = sum(out[i] for i in range(8))
    for i, n in enumerate(names):
        print(f"{n:22s} {out[i] / tot:6.3f}")


if __name__ == "__main__":
    main()
