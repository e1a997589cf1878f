"""Where the end-to-end host-buffer step's time goes (developer tool).

    python tools/e2e_breakdown.py [C3] [steps]

Prints the PCIe copy-engine rates for a field-sized pinned buffer (H2D and
D2H), the time of CsphTvdStepper.step(FlowState) on pinned arrays, and the
library's own per-bucket device times of those steps (forces, k_step with its
write-through to the host arrays)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper, scenarios as S
    from paper_1705_00614_b200.types import FlowState
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    E = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    sc = S.build(cfg, device="cuda")
    n = sc.cells()
    out = {"config": cfg, "cells": n}

    # copy-engine rates for one fp64 field
    hb = torch.empty(n, dtype=torch.float64).pin_memory()
    db = torch.empty(n, dtype=torch.float64, device="cuda")
    for name, fn in (("h2d_GBps", lambda: db.copy_(hb, non_blocking=True)),
                     ("d2h_GBps", lambda: hb.copy_(db, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        out[name] = round(3 * 8 * n / (time.perf_counter() - t0) / 1e9, 2)
    del hb, db

    st = CsphTvdStepper(sc.terrain, sc.params, sc.control, sc.options)
    if sc.wind.any():
        st.set_wind(sc.wind)
    if sc.sources:
        st.set_sources(sc.sources)
    st.upload(sc.state)
    st.run(20)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
    hs = FlowState(sc.terrain.nx, sc.terrain.ny, 0.0, pin(sc.state.H), pin(sc.state.HUx),
                   pin(sc.state.HUy))
    st.download(hs)
    st.step(hs)
    torch.cuda.synchronize()
    st.set_timing(E)
    t0 = time.perf_counter()
    for _ in range(E):
        st.step(hs)
    wall = (time.perf_counter() - t0) / E
    tk = st.timing_read(E)
    st.set_timing(0)
    na, ntot, cpt = st.active_tiles()
    out.update({
        "step_ms": round(wall * 1e3, 2),
        "ingest_bytes": st.last_ingest_bytes(),
        "writeback_bytes_upper": 3 * 8 * na * cpt,
        "bucket_ms": [round(float(tk[:, i].mean()) * 1e3, 3) for i in range(tk.shape[1])],
    })
    print(json.dumps(out))


if __name__ == "__main__":
    main()
