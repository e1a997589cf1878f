"""Generate the golden vectors in tests/golden/ from the REAL reference
(oracle/_ref/libswflood_ref.so, compiled from /root/reference by
oracle/Makefile).  Run in the build container (the reference is not on the
GPU box):   python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import pyorc  # noqa: E402
from paper_1705_00614_b200 import scenarios as S  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def digest(st):
    h = hashlib.sha256()
    for a in (st.H, st.HUx, st.HUy):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def info_dict(i):
    return {"tau": i.tau.hex(), "active_fraction": i.active_fraction.hex(),
            "lagrangian_blocks": i.lagrangian_blocks, "flux_blocks": i.flux_blocks,
            "total_blocks": i.total_blocks,
            "clamp_deficit_volume": i.clamp_deficit_volume.hex(),
            "source_volume": i.source_volume.hex(),
            "boundary_outflow_volume": i.boundary_outflow_volume.hex()}


def run_case(sc, steps, dt_cap=0.0):
    st = sc.state.copy()
    # OpenMP workers do not change the reference's bits
    sc.options.workers = os.cpu_count() or 1
    o = pyorc.OracleStepper(sc.terrain, sc.params, sc.control, sc.options, kind="ref")
    if sc.wind.any():
        o.set_wind(sc.wind)
    if sc.sources:
        o.set_sources(sc.sources)
    infos = [o.step(st, dt_cap) for _ in range(steps)]
    return st, infos


CASES = {
    # name: (factory, steps, dt_cap)
    "c1_dry_n0": (lambda: S.dam_break_1d(False, 0.0), 1000, 0.0),
    "c1_wet_n002": (lambda: S.dam_break_1d(True, 0.02), 1000, 0.0),
    "c1_dry_n002_capped": (lambda: S.dam_break_1d(False, 0.02), 500, 0.05),
    "c2_128": (lambda: S.circular_dam_break(128, 8.0, 16), 200, 0.0),
    "flood64_all_physics": (lambda: S.floodplain(64, 50.0), 60, 0.0),
    "lake128": (lambda: S.lake_at_rest(128), 200, 0.0),
}

# BASELINE.json configs at their stated sizes (VERDICT r1 "parity at the
# configs' stated sizes"): digests only (the arrays are 32-96 MB each), plus
# every step's tau.  make_golden.py --big regenerates them (several minutes).
BIG_CASES = {
    # C2: 2048^2 circular dam break, h = 8 m, n = 0.03, radius 256 cells, 1000 steps
    "c2_2048_full": (lambda: S.circular_dam_break(2048, 8.0, 256, n_manning=0.03), 1000, 0.0),
    # C3: the wettest of the bench's 8 diagonal 2048^2 crops (48.8 % wet), 200 steps
    "c3_crop2048_k5": (lambda: S.build("C3", window=(10240, 10240, 2048, 2048)), 200, 0.0),
    # C5 (h = 25 m, all physics): a 1024^2 crop with a wet/dry mix and the rain
    # source over its north-east quadrant, 200 steps
    "c5_crop1024_rain": (lambda: S.build("C5", window=(3584, 19968, 1024, 1024)), 200, 0.0),
}


def big():
    pyorc.build()
    path = os.path.join(HERE, "golden_big.json")
    out = {"generator": "tests/golden/make_golden.py --big",
           "reference": "/root/reference/proj (compiled by oracle/Makefile)", "cases": {}}
    if os.path.exists(path):
        with open(path) as f:
            out["cases"].update(json.load(f)["cases"])
    for name, (fac, steps, cap) in BIG_CASES.items():
        if name in out["cases"] and "--redo" not in sys.argv:
            continue
        sc = fac()
        import time
        t0 = time.time()
        st, infos = run_case(sc, steps, cap)
        out["cases"][name] = {"steps": steps, "dt_cap": cap, "cells": sc.cells(), "t": st.t.hex(),
                              "sha256": digest(st), "last_info": info_dict(infos[-1]),
                              "taus": [i.tau.hex() for i in infos],
                              "wet_cells_end": int((st.H > sc.params.eps_dry).sum()),
                              "ref_seconds": round(time.time() - t0, 1)}
        print(name, st.t, out["cases"][name]["sha256"][:16], f"{time.time() - t0:.1f} s", flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1)


def main():
    if "--big" in sys.argv:
        big()
        return
    pyorc.build()
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj (compiled by oracle/Makefile)",
           "cases": {}, "kat": {}}
    for name, (fac, steps, cap) in CASES.items():
        sc = fac()
        st, infos = run_case(sc, steps, cap)
        out["cases"][name] = {"steps": steps, "dt_cap": cap, "t": st.t.hex(), "sha256": digest(st),
                              "last_info": info_dict(infos[-1]),
                              "taus": [i.tau.hex() for i in infos[-5:]]}
        if name == "flood64_all_physics":
            np.savez_compressed(os.path.join(HERE, "flood64_all_physics.npz"), H=st.H, HUx=st.HUx,
                                HUy=st.HUy, t=np.array([st.t]))
        print(name, st.t, out["cases"][name]["sha256"][:16])
    # SPEC known answers evaluated by the reference's free functions
    ref = pyorc.load("ref")
    import ctypes as C
    o2 = (C.c_double * 2)()
    ref.orc_bottom_friction(1.0, 0.0, 1.0, 9.81, 0.02, o2)
    out["kat"]["friction"] = [o2[0], o2[1]]
    ref.orc_coriolis_force(1.0, 0.0, 7.292e-5, o2)
    out["kat"]["coriolis"] = [o2[0], o2[1]]
    ref.orc_wind_force(0.0, 0.0, 2.0, 5.0, 0.0, 1e-3, 1.2, 1000.0, o2)
    out["kat"]["wind"] = [o2[0], o2[1]]
    o3 = (C.c_double * 3)()
    ref.orc_hll_face_flux((C.c_double * 6)(1.0, 0.0, 0.0, 0.0, 0.0, 0.0), 9.81, o3)
    out["kat"]["hll_dam_break"] = [o3[0], o3[1], o3[2]]
    ref.orc_hll_face_flux((C.c_double * 6)(2.0, 0.0, 0.0, 2.0, 0.0, 0.0), 9.81, o3)
    out["kat"]["hll_equal_states"] = [o3[0], o3[1], o3[2]]
    out["kat"]["omega_48_7"] = ref.orc_latitude_to_omega_z(48.7)
    rng = np.random.default_rng(1705)
    xs = np.concatenate([rng.uniform(0, 1e3, 50000), 2.0 ** rng.uniform(-60, 20, 50000),
                         -rng.uniform(0, 10, 1000)])
    ys = np.array([ref.orc_cbrt(float(x)) for x in xs])
    out["kat"]["cbrt_sha256"] = hashlib.sha256(ys.tobytes()).hexdigest()
    out["kat"]["cbrt_inputs"] = "np.random.default_rng(1705): uniform(0,1e3,50000), 2**uniform(-60,20,50000), -uniform(0,10,1000)"
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
