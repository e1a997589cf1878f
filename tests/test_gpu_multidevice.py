"""The multi-GPU paths on DISTINCT devices (skipped on a one-GPU box, where
tests/test_gpu_multirank.py and tests/test_pybind.py run the same code with
the strips sharing the device): cross-device CUDA-IPC peer stores over
NVLink with NCCL between ranks, and the in-process swf_group with
cudaDeviceEnablePeerAccess between devices -- bit-identical to the
single-grid runs."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _ndev():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


needs_two = pytest.mark.skipif(_ndev() < 2, reason="needs >= 2 GPUs (distinct devices)")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@needs_two
@pytest.mark.parametrize("halo", ["p2p", "copy"])
def test_torchrun_nccl_strips_on_distinct_devices(halo):
    world = min(_ndev(), 4)
    env = dict(os.environ, SWF_DIST_BACKEND="nccl", SWF_CHECK_N="1024", SWF_CHECK_STEPS="20",
               SWF_HALO=halo)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "multirank_check.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "bitwise_equal=True" in r.stdout


@needs_two
def test_group_on_distinct_devices_matches_oracle(oracle_built):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import assert_state_bitwise, make
    from test_pybind import sw, to_native
    from paper_1705_00614_b200 import scenarios as S
    devices = min(_ndev(), 4)
    sc = S.floodplain(256, 50.0)
    T, P, K, O, W, srcs, st = to_native(sc)
    O.devices = devices
    g = sw.CsphTvdStepper(T, P, K, O)
    g.set_wind(W)
    g.set_sources(srcs)
    o = make(oracle_built.OracleStepper, sc)
    ref = sc.state.copy()
    for _ in range(10):
        a = g.step(st)
        b = o.step(ref)
        assert a.tau == b.tau
    out = sc.state.copy()
    out.H[:], out.HUx[:], out.HUy[:], out.t = st.H, st.HUx, st.HUy, st.t
    assert_state_bitwise(out, ref, f"{devices} distinct devices")
