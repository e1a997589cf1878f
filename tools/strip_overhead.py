"""Strip overhead on one GPU (developer tool): C3 stepped as P virtual strips
through the asynchronous strip path, wall time per step for P = 1, 2, 4, 8
(the strips share the device, so the totals compare per-GPU efficiency of
the strip kernels, not scaling).

    python tools/strip_overhead.py [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1705_00614_b200 import multigpu as M
    from paper_1705_00614_b200 import scenarios as S
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n = 16384
    out = {}
    for parts in (1, 2, 4, 8):
        strips = []
        for j0, j1 in M.strip_bounds(n, parts, 16):
            w0, w1 = M.window_rows(j0, j1, n)
            sc = S.build("C3", device="cuda", window=(0, w0, n, w1 - w0))
            s = M.Strip(sc, n, j0, j1, sc.global_sources, sc.wind)
            s.upload(sc.state.H, sc.state.HUx, sc.state.HUy, 0.0)
            strips.append(s)
            del sc
        M.local_steps_async(strips, 3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M.local_steps_async(strips, K)
        torch.cuda.synchronize()
        out[parts] = round((time.perf_counter() - t0) / K * 1e3, 3)
        for s in strips:
            s.close()
        del strips
        torch.cuda.empty_cache()
    print(json.dumps({"ms_per_step_by_strips": out}))


if __name__ == "__main__":
    main()
