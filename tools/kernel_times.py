"""Per-kernel device times of the fused step on a config (CUDA events on the
library stream).  SWF_LIB selects a library build.  Usage:
    python tools/kernel_times.py [C3] [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper, scenarios as S
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    sc = S.build(cfg, device="cuda")
    st = CsphTvdStepper(sc.terrain, sc.params, sc.control, sc.options)
    st.set_wind(sc.wind)
    st.set_sources(sc.sources)
    st.upload(sc.state)
    st.run(3)
    st.set_timing(K)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.run(K)
    st.sync()
    wall = (time.perf_counter() - t0) / K
    tk = st.timing_read(K).mean(axis=0)
    names = ["begin+mask", "forces", "tau", "-", "-", "-", "step", "reduce+finish"]
    out = {"lib": os.environ.get("SWF_LIB", "default"), "wall_ms": round(wall * 1e3, 3)}
    out.update({names[i]: round(tk[i] * 1e3, 3) for i in (0, 1, 2, 6, 7)})
    try:
        st.set_timing(0)
        st.step_resident()
        f, s_ = st.redo_counts()
        na, ntot, _ = st.active_tiles()
        out["redo_tiles"] = [f, s_]
        out["active_tiles"] = na
    except Exception as e:  # older library builds
        out["redo_tiles"] = str(e)[:40]
    if os.environ.get("SWF_HASH", "1") != "0":  # bitwise identity across library variants
        import hashlib
        import numpy as np
        st.sync()
        h = hashlib.sha256()
        s = sc.state
        st.download(s)
        for a in (s.H, s.HUx, s.HUy):
            a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
            h.update(np.ascontiguousarray(a).tobytes())
        h.update(repr(s.t).encode())
        out["state_sha"] = h.hexdigest()[:16]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
