"""The multi-rank strip path end to end on one GPU: torchrun with 2 and 3
ranks (gloo with host-staged halos, so several ranks can share the single
GPU of the test box), bit-identical to the single-context run."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,halo,migrate", [(2, "copy", "0"), (3, "copy", "0"), (2, "p2p", "0"),
                                               (3, "p2p", "0"), (3, "copy", "1"), (2, "p2p", "1")])
def test_torchrun_strips_bitwise(world, halo, migrate):
    """halo=p2p: k_step stores the boundary rows straight into the
    neighbours' ghost rows through CUDA IPC mappings (here several processes
    on one device; across GPUs the same stores go over NVLink).
    migrate=1: mid-run dynamic rebalancing (RankStrip.rebalance / migrate:
    rows move between ranks, the strips are rebuilt), still bitwise."""
    env = dict(os.environ, SWF_DIST_BACKEND="gloo", SWF_CHECK_N="512", SWF_CHECK_STEPS="15",
               SWF_HALO=halo, SWF_CHECK_MIGRATE=migrate)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "multirank_check.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "bitwise_equal=True" in r.stdout


def _fuzz_seeds(count, steps, world):
    """Random scenarios (tests/fuzz_scenarios.py) that split into `world`
    strips of >= 3 rows and do not abort within `steps` (checked on the CPU
    oracle), so a torchrun run of them must complete and match."""
    from fuzz_scenarios import random_scenario
    from helpers import make
    from oracle import pyorc
    from paper_1705_00614_b200 import multigpu as M
    out, seed = [], 0
    while len(out) < count and seed < 400:
        sc = random_scenario(seed)
        try:
            M.strip_bounds(sc.terrain.ny, world, sc.options.block_size)
            o = make(pyorc.OracleStepper, sc, kind="orc")
            st = sc.state.copy()
            for _ in range(steps):
                o.step(st)
            out.append(seed)
        except Exception:  # noqa: BLE001 -- too small to split, or aborts
            pass
        seed += 1
    return out


@pytest.mark.parametrize("world,halo,migrate", [(2, "copy", "0"), (3, "copy", "0"),
                                               (2, "p2p", "0"), (3, "p2p", "0"),
                                               (3, "copy", "1"), (2, "p2p", "1")])
def test_torchrun_strips_random_scenarios(oracle_built, world, halo, migrate):
    """The torchrun strip path (RankStrip: exchange, device allreduce-max,
    P2P or copy halos) on seeded random scenarios (tests/fuzz_scenarios.py:
    any block size, open / reflective edges, sources, wind): bitwise equal
    to the single grid; migrate=1 re-cuts and moves the strips mid-run."""
    seeds = _fuzz_seeds(3, 12, world)
    assert seeds
    for seed in seeds[(0 if halo == "copy" else 1):][:2]:
        env = dict(os.environ, SWF_DIST_BACKEND="gloo", SWF_CHECK_FUZZ=str(seed),
                   SWF_CHECK_STEPS="12", SWF_HALO=halo, SWF_CHECK_MIGRATE=migrate)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
               str(_port()), os.path.join(ROOT, "tests", "multirank_check.py")]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert r.returncode == 0, f"seed {seed}: " + r.stdout[-3000:] + r.stderr[-3000:]
        assert "bitwise_equal=True" in r.stdout, seed
