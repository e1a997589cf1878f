"""Host-side logic of the multi-GPU row-strip path on CPU: the strip
decomposition and the halo-exchange / allreduce protocol, run with
torch.distributed gloo at world_size 2 and 3 (same code as the NCCL path)."""
import os
import socket

import numpy as np
import pytest

from paper_1705_00614_b200 import multigpu as M


def test_strip_bounds_block_aligned_and_balanced():
    for ny, bs in ((16384, 16), (1000, 16), (96, 7), (32768, 16)):
        for parts in (1, 2, 3, 4, 8):
            b = M.strip_bounds(ny, parts, bs)
            assert b[0][0] == 0 and b[-1][1] == ny
            assert all(a[1] == c[0] for a, c in zip(b, b[1:]))
            assert all(j0 % bs == 0 for j0, _ in b)
            h = [j1 - j0 for j0, j1 in b]
            assert max(h) - min(h) < 2 * bs  # whole block rows; the last may be partial
    with pytest.raises(ValueError):
        M.strip_bounds(32, 3, 16)


def test_window_rows():
    assert M.window_rows(0, 100, 200) == (0, 103)
    assert M.window_rows(100, 200, 200) == (97, 200)
    assert M.window_rows(64, 128, 256) == (61, 131)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ny, nx, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bounds = M.strip_bounds(ny, world, 4)
        j0, j1 = bounds[rank]
        w0, w1 = M.window_rows(j0, j1, ny)
        # global field f(j, i) = 1000*j + i; each rank owns rows [j0,j1) and
        # starts with NaN ghost rows
        win = np.full((w1 - w0, nx), np.nan)
        own = np.arange(j0, j1)[:, None] * 1000.0 + np.arange(nx)[None, :]
        win[j0 - w0:j1 - w0] = own
        fields = [win.copy(), win.copy() + 0.5, win.copy() - 0.5]
        r0, r1 = j0 - w0, j1 - w0
        counts = {0: (j0 - w0) * nx, 1: (w1 - j1) * nx}

        def pack(side, t):
            rows = slice(r0, r0 + (j0 - w0)) if side == 0 else slice(r1 - (w1 - j1), r1)
            t.copy_(torch.from_numpy(np.concatenate([f[rows].reshape(-1) for f in fields])))

        def unpack(side, t):
            rows = slice(0, r0) if side == 0 else slice(r1, w1 - w0)
            n = counts[side]
            a = t.numpy()
            for k, f in enumerate(fields):
                f[rows] = a[k * n:(k + 1) * n].reshape(-1, nx)

        M.dist_exchange(pack, unpack, counts, rank, world, torch.device("cpu"))
        exp = np.arange(w0, w1)[:, None] * 1000.0 + np.arange(nx)[None, :]
        ok = all(np.array_equal(f, exp + d) for f, d in zip(fields, (0.0, 0.5, -0.5)))
        speed = M.dist_allreduce_max(float(rank) * 1.5 + 0.25, torch.device("cpu"))
        q.put((rank, ok, speed))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_exchange_and_allreduce(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 24, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, speed in res:
        assert ok, f"rank {rank}: ghost rows differ from the neighbour's owned rows"
        assert speed == (world - 1) * 1.5 + 0.25


def test_balanced_bounds_equalise_weight():
    rng = np.random.default_rng(2)
    w = rng.uniform(0.1, 1.0, 256)
    w[40:60] *= 8.0  # a busy band
    for parts in (2, 3, 5, 8):
        b = M.balanced_bounds(w, parts, 16, 256 * 16)
        assert b[0][0] == 0 and b[-1][1] == 256 * 16
        assert all(j0 % 16 == 0 and j0 < j1 for j0, j1 in b)
        assert all(b[k][1] == b[k + 1][0] for k in range(parts - 1))
        loads = [w[j0 // 16:j1 // 16].sum() for j0, j1 in b]
        assert max(loads) / (sum(loads) / parts) < 1.0 + 2 * w.max() * parts / w.sum()
    eq = M.balanced_bounds(np.ones(64), 4, 16, 1024)
    assert eq == M.strip_bounds(1024, 4, 16)


def test_weak_scaling_sources_clipped_to_the_band():
    """C5W (weak scaling) keeps the C5 generator's first 4096*N rows; its
    sources are clipped to them (scenarios.clip_sources)."""
    from paper_1705_00614_b200 import scenarios as S
    from paper_1705_00614_b200.types import CellRect, SourceKind, SourceSpec, Vec2
    specs = [SourceSpec(SourceKind.Discharge, "a", CellRect(1, 10, 4, 20), [], 0.0, Vec2()),
             SourceSpec(SourceKind.Rain, "b", CellRect(5, 4090, 9, 5000), [], 1e-6, Vec2()),
             SourceSpec(SourceKind.Rain, "c", CellRect(5, 9000, 9, 9100), [], 1e-6, Vec2())]
    out = S.clip_sources(specs, 32768, 4096)
    assert [s.name for s in out] == ["a", "b"]
    assert (out[1].cells.j0, out[1].cells.j1) == (4090, 4095)
    assert S.WEAK_ROWS == 4096


def test_transfer_plan_covers_every_new_window_once():
    for ny, parts in ((256, 2), (512, 3), (1024, 5)):
        old = M.strip_bounds(ny, parts, 16)
        rng = np.random.default_rng(parts)
        w = rng.uniform(0.1, 5.0, ny // 16)
        new = M.balanced_bounds(w, parts, 16, ny)
        plan = M.transfer_plan(old, new, ny)
        for dst, (j0, j1) in enumerate(new):
            w0, w1 = M.window_rows(j0, j1, ny)
            got = np.zeros(ny, int)
            for src, d, a, b in plan:
                if d == dst:
                    o0, o1 = old[src]
                    assert o0 <= a < b <= o1  # a source sends rows it owns
                    got[a:b] += 1
            assert (got[w0:w1] == 1).all() and got.sum() == w1 - w0


def test_rebalance_bounds_decision():
    ny, bs = 512, 16
    w = np.ones(ny // bs)
    b = M.strip_bounds(ny, 4, bs)
    assert M.rebalance_bounds(w, b, bs, ny) is None  # already balanced
    w2 = w.copy()
    w2[:8] = 20.0  # the flood front moved into the first strip
    new = M.rebalance_bounds(w2, b, bs, ny)
    assert new is not None
    assert max(M.strip_loads(w2, new, bs)) < max(M.strip_loads(w2, b, bs))
    assert new[0][0] == 0 and new[-1][1] == ny and all(j0 % bs == 0 for j0, _ in new)
    # a marginal gain below the threshold keeps the strips
    w3 = w.copy()
    w3[0] = 1.01
    assert M.rebalance_bounds(w3, b, bs, ny, threshold=0.05) is None


def test_strip_bounds_every_strip_owns_a_full_halo():
    """Every strip of a multi-strip split owns >= HALO rows (a neighbour's
    ghost rows all come from one strip; swf_create_strip rejects smaller
    strips), block-aligned cuts tile the grid, for the even and the
    activity-balanced split alike; impossible splits raise ValueError."""
    import random
    from paper_1705_00614_b200 import multigpu as M
    rnd = random.Random(1705)
    seen = 0
    for _ in range(5000):
        ny = rnd.randint(1, 300)
        bs = rnd.choice([1, 2, 3, 4, 7, 8, 16, 32])
        parts = rnd.randint(1, 9)
        nbr = (ny + bs - 1) // bs
        for kind in ("even", "balanced"):
            try:
                if kind == "even":
                    b = M.strip_bounds(ny, parts, bs)
                else:
                    w = [rnd.random() ** 4 for _ in range(nbr)]
                    b = M.balanced_bounds(w, parts, bs, ny)
            except ValueError:
                assert parts > 1
                continue
            seen += 1
            assert len(b) == parts and b[0][0] == 0 and b[-1][1] == ny
            for (a0, a1), (c0, c1) in zip(b, b[1:]):
                assert a1 == c0 and c0 % bs == 0
            if parts > 1:
                assert all(j1 - j0 >= M.HALO for j0, j1 in b), (ny, bs, parts, b)
    assert seen > 5000
    assert M.strip_bounds(33, 2, 16) == [(0, 16), (16, 33)]
