"""Run under torchrun: N ranks each own a row strip of a floodplain, step it
through the same RankStrip code the multi-GPU bench uses (exchange + exact
allreduce-max), gather on rank 0 and compare bit for bit with a single
context stepping the whole grid.  Exit code 0 = identical."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch.distributed as dist
    from paper_1705_00614_b200 import CsphTvdStepper, multigpu as M, scenarios as S
    n = int(os.environ.get("SWF_CHECK_N", "512"))
    steps = int(os.environ.get("SWF_CHECK_STEPS", "20"))
    fuzz = os.environ.get("SWF_CHECK_FUZZ")  # a seed of tests/fuzz_scenarios.py
    if fuzz is not None:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from fuzz_scenarios import random_scenario
        full = random_scenario(int(fuzz))
        rs = M.RankStrip("custom", scenario=full)
        n = full.terrain.nx
    else:
        full = None
        rs = M.RankStrip("C3", n_full=n)
    p2p = os.environ.get("SWF_HALO") == "p2p"
    if p2p:
        assert rs.setup_p2p(), "P2P halo setup failed"
    migrate = os.environ.get("SWF_CHECK_MIGRATE") == "1"
    for k in range(steps):
        if migrate and k == steps // 3:
            # dynamic rebalancing: re-cut from the current activity (any change
            # accepted), then force a move of every interior cut by a block row
            rs.rebalance(threshold=-1.0)
            b = [list(x) for x in rs.bounds]
            bs = rs.bs
            keep = max(bs, M.HALO)  # a block row, and at least the halo, stays on each side
            for q in range(1, rs.world):
                d = bs if q % 2 else -bs
                if b[q - 1][0] + keep <= b[q][0] + d <= b[q][1] - keep:
                    b[q - 1][1] = b[q][0] = b[q][0] + d
            rs.migrate([tuple(x) for x in b])
        if p2p:
            rs.step_p2p()
        else:
            rs.step()
    got = rs.gather_state()
    ok = 1
    if rs.rank == 0:
        if full is None:
            full = S.floodplain(n, 50.0, device="cuda")
        one = CsphTvdStepper(full.terrain, full.params, full.control, full.options)
        if full.wind.any():
            one.set_wind(full.wind)
        if full.sources:
            one.set_sources(full.sources)
        st = full.state.copy()
        one.upload(st)
        one.run(steps)
        one.download(st)
        (H, X, Y), t = got
        same = all(np.array_equal(a.view(np.int64), b.view(np.int64))
                   for a, b in ((H, st.H), (X, st.HUx), (Y, st.HUy))) and t == st.t
        print(f"multirank world={rs.world} n={n} steps={steps} p2p={p2p} migrate={migrate} "
              f"bounds={rs.bounds} bitwise_equal={same} t={t}",
              flush=True)
        ok = 1 if same else 0
    flag = [ok]
    dist.broadcast_object_list(flag, src=0)
    dist.destroy_process_group()
    sys.exit(0 if flag[0] else 1)


if __name__ == "__main__":
    main()
