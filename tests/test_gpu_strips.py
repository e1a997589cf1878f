"""Row strips on ONE GPU (virtual ranks): P strip contexts exchanging halos
through the same pack/unpack entry points the NCCL path uses, against the
single-grid run.  Bit-identical by construction (exact max-reduction of the
CFL speed, unchanged per-cell arithmetic)."""
import numpy as np
import pytest

from helpers import assert_bitwise, make
from paper_1705_00614_b200 import multigpu as M
from paper_1705_00614_b200 import scenarios as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("parts,mode", [(2, "sync"), (3, "sync"), (4, "sync"), (2, "async"),
                                        (3, "async"), (5, "async")])
def test_strips_bitwise_equal_single_grid(parts, mode):
    from paper_1705_00614_b200 import CsphTvdStepper
    n = 256
    full = S.floodplain(n, 50.0)
    one = make(CsphTvdStepper, full)
    st = full.state.copy()
    one.upload(st)
    one.run(25)
    one.download(st)
    bounds = M.strip_bounds(n, parts, full.options.block_size)
    strips = []
    for j0, j1 in bounds:
        w0, w1 = M.window_rows(j0, j1, n)
        sc = S.floodplain(n, 50.0, window=(0, w0, n, w1 - w0))
        s = M.Strip(sc, n, j0, j1, sc.global_sources, sc.wind)
        s.upload(sc.state.H, sc.state.HUx, sc.state.HUy, 0.0)
        strips.append((s, sc, w0))
    if mode == "sync":
        for _ in range(25):
            M.local_step([s for s, _, _ in strips])
    else:  # interior forces / exchange / boundary forces / device allreduce
        res = M.local_steps_async([s for s, _, _ in strips], 25)
        assert all(done == 25 for done, _ in res)
    H = np.empty(n * n)
    X = np.empty(n * n)
    Y = np.empty(n * n)
    t = None
    for (s, sc, w0), (j0, j1) in zip(strips, bounds):
        h = np.empty_like(sc.state.H)
        x = np.empty_like(h)
        y = np.empty_like(h)
        t = s.download(h, x, y)
        r0 = (j0 - w0) * n
        H[j0 * n:j1 * n] = h[r0:r0 + (j1 - j0) * n]
        X[j0 * n:j1 * n] = x[r0:r0 + (j1 - j0) * n]
        Y[j0 * n:j1 * n] = y[r0:r0 + (j1 - j0) * n]
    assert t == st.t
    assert_bitwise(H, st.H, "H")
    assert_bitwise(X, st.HUx, "HUx")
    assert_bitwise(Y, st.HUy, "HUy")


@pytest.mark.parametrize("parts", [2, 3])
def test_strip_host_steps_from_pinned_windows(parts):
    """The strips' host-buffer step (swf_strip_host_phase1/2): every strip
    reads its window from ONE pinned global state (depth in full, momentum of
    its flux-active tiles and ghost rows), the speeds are max-reduced, and
    each k_step writes its owned cells back in place -- bit-identical to the
    single-grid run."""
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper
    n = 256
    full = S.floodplain(n, 50.0)
    one = make(CsphTvdStepper, full)
    ref = full.state.copy()
    one.upload(ref)
    one.run(12)
    one.download(ref)
    pin = lambda a: torch.from_numpy(np.array(a, copy=True)).pin_memory().numpy()
    H, X, Y = pin(full.state.H), pin(full.state.HUx), pin(full.state.HUy)
    bounds = M.strip_bounds(n, parts, full.options.block_size)
    strips = []
    for j0, j1 in bounds:
        w0, w1 = M.window_rows(j0, j1, n)
        sc = S.floodplain(n, 50.0, window=(0, w0, n, w1 - w0))
        strips.append((M.Strip(sc, n, j0, j1, sc.global_sources, sc.wind), w0 * n))
    t = 0.0
    for _ in range(12):
        sp = [s.host_phase1(H[o:], X[o:], Y[o:], t) for s, o in strips]
        g = max(sp)
        ts = [s.host_phase2(H[o:], X[o:], Y[o:], g)[0] for s, o in strips]
        assert len(set(ts)) == 1
        t = ts[0]
        assert all(s.last_ingest_bytes() < 3 * 8 * H.size for s, _ in strips)
    assert t == ref.t
    assert_bitwise(H, ref.H, "H")
    assert_bitwise(X, ref.HUx, "HUx")
    assert_bitwise(Y, ref.HUy, "HUy")


def test_strip_owning_fewer_rows_than_the_halo_is_rejected():
    """A neighbour's 3 ghost rows must come from one strip's owned rows:
    swf_create_strip refuses a smaller strip with a ConfigError (and the
    splits never produce one, tests/test_multigpu_cpu.py)."""
    from paper_1705_00614_b200 import ConfigError
    n = 64
    def window(j0, j1):
        w0, w1 = M.window_rows(j0, j1, n)
        sc = S.floodplain(n, 50.0, window=(0, w0, n, w1 - w0))
        sc.options.block_size = 1  # (strip cuts are block-aligned)
        return sc

    for j0, j1 in ((30, 32), (0, 2), (62, 64)):
        sc = window(j0, j1)
        with pytest.raises(ConfigError, match="at least 3 rows"):
            M.Strip(sc, n, j0, j1, sc.global_sources, sc.wind)
    sc = window(29, 32)  # exactly the halo depth is fine
    M.Strip(sc, n, 29, 32, sc.global_sources, sc.wind).close()
