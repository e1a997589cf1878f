"""A numerical abort in ONE row strip of a multi-step batch commits the same
step count on every strip (swf_group_run with nsteps > 1, and the
asynchronous strip batch).  The failing strip stops at once; the others are
stopped in the next step before their K4..K8 (k_group_max / the stop marker
in the int64 speed allreduce), and the ones that finished one step more roll
it back (swf_strip_settle).  The committed state must be the step-start
state, bit for bit, with the reference's error message."""
import ctypes as C

import numpy as np
import pytest

from helpers import assert_bitwise, make
from paper_1705_00614_b200 import multigpu as M
from paper_1705_00614_b200 import scenarios as S

pytestmark = pytest.mark.gpu

N = 256


def _poisoned():
    """C3-like floodplain with a NaN momentum in one wet cell well inside
    the upper strip (the reference aborts with a non-finite face flux)."""
    full = S.floodplain(N, 50.0)
    st = full.state.copy()
    H = st.H.reshape(N, N)
    rows = np.arange(N)[:, None] * np.ones((1, N), dtype=int)
    cand = np.flatnonzero((H > 0.5).ravel() & (rows.ravel() > 200) & (rows.ravel() < 240))
    k = int(cand[len(cand) // 2])
    st.HUx[k] = np.nan
    return full, st


def _strips(full, st, parts):
    bounds = M.strip_bounds(N, parts, full.options.block_size)
    out = []
    for j0, j1 in bounds:
        w0, w1 = M.window_rows(j0, j1, N)
        sc = S.floodplain(N, 50.0, window=(0, w0, N, w1 - w0))
        s = M.Strip(sc, N, j0, j1, sc.global_sources, sc.wind)
        sl = slice(w0 * N, w1 * N)
        s.upload(st.H[sl].copy(), st.HUx[sl].copy(), st.HUy[sl].copy(), st.t)
        out.append((s, sc, w0, j0, j1))
    return out


def _gather(strips):
    H, X, Y = (np.empty(N * N) for _ in range(3))
    ts = set()
    for s, sc, w0, j0, j1 in strips:
        h, x, y = (np.empty_like(sc.state.H) for _ in range(3))
        ts.add(s.download(h, x, y))
        r0 = (j0 - w0) * N
        n = (j1 - j0) * N
        H[j0 * N:j1 * N], X[j0 * N:j1 * N], Y[j0 * N:j1 * N] = h[r0:r0 + n], x[r0:r0 + n], y[r0:r0 + n]
    return H, X, Y, ts


def _oracle_message(oracle_built, full, st):
    from paper_1705_00614_b200 import NumericalError
    o = make(oracle_built.OracleStepper, full, kind="orc")
    with pytest.raises(NumericalError) as eo:
        o.step(st.copy())
    return str(eo.value)


@pytest.mark.parametrize("parts", [2, 3])
def test_async_batch_abort_in_one_strip(oracle_built, parts):
    from paper_1705_00614_b200 import NumericalError
    full, st = _poisoned()
    msg = _oracle_message(oracle_built, full, st)
    strips = _strips(full, st, parts)
    with pytest.raises(NumericalError) as eg:
        M.local_steps_async([s for s, *_ in strips], 4)
    assert str(eg.value) == msg
    assert all(s.steps_done() == 0 for s, *_ in strips)
    H, X, Y, ts = _gather(strips)
    assert ts == {st.t}
    assert_bitwise(H, st.H, "H")
    assert_bitwise(X, st.HUx, "HUx")
    assert_bitwise(Y, st.HUy, "HUy")
    # the strips keep working from the committed state: a clean state steps on
    good = full.state.copy()
    for s, sc, w0, j0, j1 in strips:
        sl = slice(w0 * N, (w0 + sc.terrain.ny) * N)
        s.upload(good.H[sl].copy(), good.HUx[sl].copy(), good.HUy[sl].copy(), good.t)
    res = M.local_steps_async([s for s, *_ in strips], 3)
    assert all(d == 3 for d, _ in res)


def test_group_run_abort_in_one_strip(oracle_built):
    from paper_1705_00614_b200._lib import lib
    full, st = _poisoned()
    msg = _oracle_message(oracle_built, full, st)
    strips = _strips(full, st, 2)
    L = lib()
    arr = (C.c_void_p * 2)(*[s.ctx for s, *_ in strips])
    g = C.c_void_p()
    assert L.swf_group_create(arr, 2, C.byref(g)) == 0
    try:
        done = C.c_int(-1)
        rc = L.swf_group_run(g, 4, 0.0, C.byref(done), None)
        assert rc == 2, rc  # SWF_ENUMERICAL
        assert done.value == 0
        assert L.swf_group_last_error(g).decode() == msg
    finally:
        L.swf_group_destroy(g)
    H, X, Y, ts = _gather(strips)
    assert ts == {st.t}
    assert_bitwise(H, st.H, "H")
    assert_bitwise(X, st.HUx, "HUx")
    assert_bitwise(Y, st.HUy, "HUy")
