"""A small workload over every kernel family, for compute-sanitizer
(developer tool):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

Fused resident steps, a pinned host-buffer step, the staged path, row strips
(synchronous and asynchronous protocol), the single-process device group, a
nested coupled step and the speculative-division redo path, each on a small
grid."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper, scenarios as S
    from paper_1705_00614_b200 import multigpu as M
    from paper_1705_00614_b200.nesting import NestedGrid, coupled_step
    from paper_1705_00614_b200.types import FlowState

    def make(sc, mode=0):
        st = CsphTvdStepper(sc.terrain, sc.params, sc.control, sc.options)
        if sc.wind.any():
            st.set_wind(sc.wind)
        if sc.sources:
            st.set_sources(sc.sources)
        if mode:
            st.set_mode(mode)
        return st

    sc = S.floodplain(96, 50.0)
    # fused resident steps + speculative redo (subnormal momenta)
    st = sc.state.copy()
    wet = np.flatnonzero(st.H > 1e-3)
    st.HUx[wet[::7]] = 3e-310
    g = make(sc)
    g.upload(st)
    g.run(3)
    g.download(st)
    # pinned host-buffer step
    pin = lambda a: torch.from_numpy(a.copy()).pin_memory().numpy()
    hs = FlowState(st.nx, st.ny, st.t, pin(st.H), pin(st.HUx), pin(st.HUy))
    g.step(hs)
    g.step(hs)
    # opt-in host mirror: the upload step, then steps without ingest
    g.set_host_mirror(True)
    for _ in range(3):
        g.step(hs)
    g.set_host_mirror(False)
    # staged path
    s2 = make(sc, mode=1)
    s2.step(sc.state.copy())
    # strips: synchronous and asynchronous protocol
    n = 128
    full = S.floodplain(n, 50.0)
    strips = []
    for j0, j1 in M.strip_bounds(n, 3, full.options.block_size):
        w0, w1 = M.window_rows(j0, j1, n)
        w = S.floodplain(n, 50.0, window=(0, w0, n, w1 - w0))
        s = M.Strip(w, n, j0, j1, w.global_sources, w.wind)
        s.upload(w.state.H, w.state.HUx, w.state.HUy, 0.0)
        strips.append(s)
    for _ in range(2):
        M.local_step(strips)
    M.local_steps_async(strips, 2)
    # a random scenario (tests/fuzz_scenarios.py: block size 7, open edges,
    # sources, wind) in 2 strips through the asynchronous protocol
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from fuzz_scenarios import random_scenario, window
    rs = random_scenario(3)
    rs.options.block_size = 7
    ny = rs.terrain.ny
    rstrips = []
    for j0, j1 in M.strip_bounds(ny, 2, 7):
        w0, w1 = M.window_rows(j0, j1, ny)
        ws = window(rs, w0, w1)
        s = M.Strip(ws, ny, j0, j1, ws.global_sources, ws.wind)
        s.upload(ws.state.H, ws.state.HUx, ws.state.HUy, 0.0)
        rstrips.append(s)
    M.local_steps_async(rstrips, 2)
    # single-process device group (pybind module over the C++ drop-in)
    try:
        from paper_1705_00614_b200 import swflood_native as sw
        T = sw.Terrain(n, n, 50.0, 0.0, 0.0, full.terrain.b)
        P = sw.PhysicalParams()
        P.n_manning = 0.03
        O = sw.StepperOptions()
        O.devices = 2
        gg = sw.CsphTvdStepper(T, P, sw.TimestepControl(), O)
        fs = sw.FlowState.dry(T)
        fs.H[:] = full.state.H
        gg.step(fs)
        gg.step(fs)
        O.block_size = 7  # the unsplit phase 1 of a block size not dividing 16
        gg = sw.CsphTvdStepper(T, P, sw.TimestepControl(), O)
        fs = sw.FlowState.dry(T)
        fs.H[:] = full.state.H
        gg.step(fs)
    except ImportError:
        pass
    # nested coupled step
    ns = S.nested_floodplain(64, 50.0, (20, 20, 16, 16), 4, 2)
    coarse = make(ns.coarse)
    coarse.upload(ns.coarse.state)
    nest = NestedGrid(coarse, ns.window, ns.r, ns.fine.terrain, ns.fine.params,
                      ns.fine.control, ns.fine.options, ghost=ns.ghost, two_way=True)
    nest.upload(ns.fine.state)
    for _ in range(2):
        coupled_step(coarse, [nest])
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
