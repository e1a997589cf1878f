"""Exploratory strip-path sweep (developer tool): random scenarios
(tests/fuzz_scenarios.py) split into 2-4 row strips on the one visible GPU,
stepped through the synchronous or the asynchronous strip protocol, against
the single-grid CUDA path (itself bitwise to the reference).
    python tools/fuzz_strips.py FIRST COUNT [STEPS]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from fuzz_scenarios import random_scenario, window  # noqa: E402
from helpers import assert_bitwise, make  # noqa: E402


def main():
    from paper_1705_00614_b200 import CsphTvdStepper
    from paper_1705_00614_b200 import multigpu as M
    first, count = int(sys.argv[1]), int(sys.argv[2])
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    t0 = time.time()
    stats = {"ok": 0, "failed": 0, "skipped_abort": 0, "skipped_config": 0}
    for seed in range(first, first + count):
        sc = random_scenario(seed)
        n_y, bs = sc.terrain.ny, sc.options.block_size
        rng = np.random.default_rng(seed)
        parts = int(rng.integers(2, 5))
        mode = "async" if seed % 2 else "sync"
        one = make(CsphTvdStepper, sc)
        st = sc.state.copy()
        one.upload(st)
        try:
            done, _ = one.run(steps)
        except Exception:
            done = -1
        if done != steps:
            stats["skipped_abort"] += 1
            continue
        one.download(st)
        try:
            bounds = M.strip_bounds(n_y, parts, bs)
            strips = []
            for j0, j1 in bounds:
                w0, w1 = M.window_rows(j0, j1, n_y)
                ws = window(sc, w0, w1)
                s = M.Strip(ws, n_y, j0, j1, ws.global_sources, ws.wind)
                s.upload(ws.state.H, ws.state.HUx, ws.state.HUy, 0.0)
                strips.append((s, ws, w0))
        except Exception as e:  # noqa: BLE001
            stats["skipped_config"] += 1
            print(json.dumps({"seed": seed, "config": str(e)[:200]}), flush=True)
            continue
        try:
            if mode == "sync":
                for _ in range(steps):
                    M.local_step([s for s, _, _ in strips])
            else:
                res = M.local_steps_async([s for s, _, _ in strips], steps)
                assert all(d == steps for d, _ in res), res
            nx = sc.terrain.nx
            for f in ("H", "HUx", "HUy"):
                full = np.empty(nx * n_y)
                for (s, ws, w0), (j0, j1) in zip(strips, bounds):
                    h = np.empty(ws.terrain.nx * ws.terrain.ny)
                    x = np.empty_like(h)
                    y = np.empty_like(h)
                    t = s.download(h, x, y)
                    assert t == st.t, (t, st.t)
                    a = {"H": h, "HUx": x, "HUy": y}[f]
                    r0 = (j0 - w0) * nx
                    full[j0 * nx:j1 * nx] = a[r0:r0 + (j1 - j0) * nx]
                assert_bitwise(full, getattr(st, f), f"seed {seed} {f}")
            stats["ok"] += 1
        except Exception as e:  # noqa: BLE001 -- a mismatch or a runtime failure
            stats["failed"] += 1
            print(json.dumps({"seed": seed, "parts": parts, "mode": mode, "bs": bs,
                              "error": str(e)[:300]}), flush=True)
        finally:
            for s, _, _ in strips:
                s.close()
    stats.update(seeds=count, first=first, steps=steps, seconds=round(time.time() - t0, 1))
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
