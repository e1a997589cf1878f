"""Row-strip decomposition of the CSPH-TVD step across GPUs.

The global nx x ny grid is cut into contiguous row strips whose boundaries
are multiples of the block size B, so every B-block (and with it the K1
activity mask and the dry-block skipping) lives on exactly one strip.  Each
strip keeps SWF_HALO = 3 ghost rows per interior side — the radius of the
step's dependency diamond — and per step:

  1. halo exchange: the 3 owned boundary rows of (H, HUx, HUy) go to each
     neighbour's ghost rows (NCCL send/recv over NVLink, or in-process
     device copies for virtual ranks);
  2. phase 1 on every strip: sources, K1 mask, K2 forces on the owned rows
     plus 2 ghost rows, and the strip's CFL speed;
  3. allreduce-MAX of the speed — exact in any order, so tau is bit-equal to
     the single-grid tau;
  4. phase 2: tau, fused K4..K8 on the owned rows.

Per-cell arithmetic is unchanged, so a P-strip run is bit-identical to the
single-grid run (tests/test_gpu_strips.py checks this on one GPU with virtual
ranks; tests/test_multigpu_cpu.py checks the exchange protocol with gloo).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi as A

HALO = 3


def min_rows_cuts(cuts, bs: int, ny: int, halo: int = HALO) -> List[int]:
    """Block-row cuts adjusted so that every strip of a multi-strip split owns
    at least `halo` rows: a neighbour's ghost rows must all come from one
    strip's owned rows (swf_create_strip rejects smaller strips).  Later strips
    grow first (the last block row may be partial), then earlier ones;
    ValueError if the grid is too small for that many strips."""
    cuts = list(cuts)
    parts = len(cuts) - 1
    if parts <= 1:
        return cuts
    rows = lambda p: min(cuts[p + 1] * bs, ny) - min(cuts[p] * bs, ny)
    for p in range(parts - 1, 0, -1):
        while rows(p) < halo and cuts[p] - 1 > cuts[p - 1]:
            cuts[p] -= 1
    for p in range(parts - 1):
        while rows(p) < halo and cuts[p + 1] + 1 < cuts[p + 2]:
            cuts[p + 1] += 1
    if any(rows(p) < halo for p in range(parts)):
        raise ValueError(f"cannot split {ny} rows into {parts} strips of at least {halo} rows "
                         f"at block size {bs}")
    return cuts


def strip_bounds(ny: int, parts: int, bs: int) -> List[Tuple[int, int]]:
    """Owned global rows [j0, j1) per strip: balanced whole block rows, every
    strip at least HALO rows (min_rows_cuts)."""
    nbr = (ny + bs - 1) // bs
    if parts < 1 or parts > nbr:
        raise ValueError(f"cannot split {nbr} block rows into {parts} strips")
    base, rem = divmod(nbr, parts)
    cuts = [0]
    for p in range(parts):
        cuts.append(cuts[-1] + base + (1 if p < rem else 0))
    cuts = min_rows_cuts(cuts, bs, ny)
    return [(cuts[p] * bs, min(cuts[p + 1] * bs, ny)) for p in range(parts)]


def balanced_bounds(weights, parts: int, bs: int, ny: int) -> List[Tuple[int, int]]:
    """Owned rows [j0, j1) per strip, cut at block-row boundaries so that the
    strips carry about equal total weight (weights: one value per block row,
    e.g. its active cells plus a small cost per dry cell).  Deterministic, so
    every rank derives the same cut from the same weights."""
    w = np.asarray(weights, dtype=np.float64)
    nbr = w.size
    if parts < 1 or parts > nbr:
        raise ValueError(f"cannot split {nbr} block rows into {parts} strips")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for p in range(1, parts):
        target = cum[-1] * p / parts
        b = int(np.searchsorted(cum, target))
        # the nearer of the two block-row boundaries around the target, keeping
        # at least one block row per strip
        if b > 0 and abs(cum[b - 1] - target) <= abs(cum[min(b, nbr)] - target):
            b -= 1
        b = max(b, cuts[-1] + 1)
        b = min(b, nbr - (parts - p))
        cuts.append(b)
    cuts.append(nbr)
    cuts = min_rows_cuts(cuts, bs, ny)
    return [(cuts[p] * bs, min(cuts[p + 1] * bs, ny)) for p in range(parts)]


def row_weights(config: str, n: int, bs: int, device: str = "cuda", dry_cost: float = 0.1):
    """Per-block-row cost of the initial state of a floodplain config: wet
    cells (their tiles run the whole step) plus dry_cost per dry cell (the
    work-list and skip bookkeeping), from the full-resolution generator."""
    from . import scenarios as S
    h = {"C3": 50.0, "C5": 25.0}[config]
    out = np.zeros((n + bs - 1) // bs)
    step = max(bs, (1 << 22) // max(n, 1) // bs * bs)  # row chunks of ~4M cells
    for j0 in range(0, n, step):
        nj = min(step, n - j0)
        sc = S.floodplain(n, h, window=(0, j0, n, nj), device=device)
        wet = (sc.state.H.reshape(nj, n) > sc.params.eps_dry).sum(axis=1)
        cost = wet + dry_cost * (n - wet)
        for r in range(nj):
            out[(j0 + r) // bs] += cost[r]
    return out


def strip_loads(weights, bounds, bs: int) -> List[float]:
    """Total weight per strip (weights: one value per block row)."""
    w = np.asarray(weights, dtype=np.float64)
    return [float(w[j0 // bs:(j1 + bs - 1) // bs].sum()) for j0, j1 in bounds]


def rebalance_bounds(weights, bounds, bs: int, ny: int, threshold: float = 0.03):
    """Dynamic strip rebalancing (the flood front migrates, so
    strips balanced at t = 0 drift out of balance): new block-row cuts from
    the current activity, or None when they would not lower the busiest
    strip's load by more than `threshold` (relative).  Deterministic: every
    rank derives the same answer from the same allgathered weights."""
    new = balanced_bounds(weights, len(bounds), bs, ny)
    if [tuple(b) for b in new] == [tuple(b) for b in bounds]:
        return None
    old_max, new_max = max(strip_loads(weights, bounds, bs)), max(strip_loads(weights, new, bs))
    return new if new_max < old_max * (1.0 - threshold) else None


def transfer_plan(old, new, ny: int, halo: int = HALO):
    """The row moves of a re-partition: (src, dst, a, b) -- rank src sends its
    owned global rows [a, b) to rank dst, which needs them in its new window
    (owned rows plus ghost rows).  Every row of every new window comes from
    exactly one owner (the old strips tile the grid)."""
    out = []
    for dst, (j0, j1) in enumerate(new):
        w0, w1 = window_rows(j0, j1, ny, halo)
        for src, (o0, o1) in enumerate(old):
            a, b = max(w0, o0), min(w1, o1)
            if a < b:
                out.append((src, dst, a, b))
    return out


def window_rows(j0: int, j1: int, ny: int, halo: int = HALO) -> Tuple[int, int]:
    """Global rows of a strip's local window (owned + ghost rows)."""
    return max(j0 - halo, 0), min(j1 + halo, ny)


class Strip:
    """One strip context of libswflood_cuda (swf_create_strip)."""

    def __init__(self, sc_window, ny_global: int, j0: int, j1: int, sources, wind,
                 device: int = 0):
        from ._lib import lib
        from ._marshal import Marshalled
        from .stepper import raise_for
        self._lib = lib()
        self._raise = raise_for
        T = sc_window.terrain
        self.nx, self.ny, self.j0, self.j1 = T.nx, ny_global, j0, j1
        self.w0, self.w1 = window_rows(j0, j1, ny_global)
        if T.ny != self.w1 - self.w0:
            raise ValueError("scenario window does not match the strip window")
        m = Marshalled()
        b = m.arr(T.b)
        t = A.swf_terrain(T.nx, ny_global, T.h, T.x0, T.y0 - self.w0 * T.h, A.dptr(b))
        p = m.params(sc_window.params, T.nx * T.ny)
        k = m.control(sc_window.control)
        o = m.options(sc_window.options)
        ctx = C.c_void_p()
        rc = self._lib.swf_create_strip(C.byref(t), C.byref(p), C.byref(k), C.byref(o), j0, j1,
                                        device, C.byref(ctx))
        raise_for(rc, None)
        self.ctx = ctx
        if wind is not None and wind.any():
            n, tt, x, y = m.wind(wind)
            self._rc(self._lib.swf_set_wind(ctx, n, tt, x, y))
        if sources:
            arr = m.sources(sources)
            self._rc(self._lib.swf_set_sources(ctx, len(sources), arr))
        self.count = {s: self._count(s) for s in (0, 1)}

    def _rc(self, rc):
        self._raise(rc, self.ctx)

    def _count(self, side):
        s3, r3 = (A.PD * 3)(), (A.PD * 3)()
        n = C.c_size_t()
        self._rc(self._lib.swf_strip_halo_ptrs(self.ctx, side, s3, r3, C.byref(n)))
        return n.value

    def close(self):
        if getattr(self, "ctx", None):
            self._lib.swf_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, H, HUx, HUy, t: float):
        self._rc(self._lib.swf_upload_state(self.ctx, A.dptr(H), A.dptr(HUx), A.dptr(HUy), t))

    def download(self, H, HUx, HUy) -> float:
        t = C.c_double()
        self._rc(self._lib.swf_download_state(self.ctx, A.dptr(H), A.dptr(HUx), A.dptr(HUy),
                                              C.byref(t)))
        return t.value

    def pack(self, side: int, dev_ptr: int):
        self._rc(self._lib.swf_strip_pack(self.ctx, side, C.c_void_p(dev_ptr)))

    def unpack(self, side: int, dev_ptr: int):
        self._rc(self._lib.swf_strip_unpack(self.ctx, side, C.c_void_p(dev_ptr)))

    def phase1(self, dt_cap: float = 0.0) -> float:
        s = C.c_double()
        self._rc(self._lib.swf_strip_phase1(self.ctx, float(dt_cap), C.byref(s)))
        return s.value

    def phase2(self, speed: float, dt_cap: float = 0.0):
        from ._marshal import info_from_c
        info = A.swf_step_info()
        self._rc(self._lib.swf_strip_phase2(self.ctx, float(speed), float(dt_cap), C.byref(info)))
        return info_from_c(info)

    # host-buffer step from pinned window arrays (include/swf.h)
    def host_phase1(self, H, HUx, HUy, t: float, dt_cap: float = 0.0) -> float:
        """H/HUx/HUy: pinned arrays whose first element is the window's first
        cell (views into a pinned global array are fine)."""
        s = C.c_double()
        tt = C.c_double(t)
        self._rc(self._lib.swf_strip_host_phase1(
            self.ctx, H.ctypes.data, HUx.ctypes.data, HUy.ctypes.data, C.byref(tt),
            float(dt_cap), C.byref(s)))
        return s.value

    def host_phase2(self, H, HUx, HUy, speed: float, dt_cap: float = 0.0):
        from ._marshal import info_from_c
        info = A.swf_step_info()
        t = C.c_double()
        self._rc(self._lib.swf_strip_host_phase2(
            self.ctx, H.ctypes.data, HUx.ctypes.data, HUy.ctypes.data, C.byref(t), float(speed),
            float(dt_cap), C.byref(info)))
        return t.value, info_from_c(info)

    def last_ingest_bytes(self) -> int:
        v = C.c_longlong()
        self._rc(self._lib.swf_last_ingest_bytes(self.ctx, C.byref(v)))
        return v.value

    def active_tiles(self):
        """(flux-active tiles, tiles, cells per tile) of the last step."""
        a, n, c = C.c_int(), C.c_int(), C.c_int()
        self._rc(self._lib.swf_active_tiles(self.ctx, C.byref(a), C.byref(n), C.byref(c)))
        return a.value, n.value, c.value

    def stream_handle(self) -> int:
        return self._lib.swf_stream(self.ctx) or 0

    def mask(self):
        """(interior, halo) block counts of the owned block rows (last step),
        shaped (block rows, nbx)."""
        a, b = C.c_int(), C.c_int()
        # the shape first (any block size), then the counts into arrays of it
        self._rc(self._lib.swf_download_mask(self.ctx, None, None, C.byref(a), C.byref(b)))
        n = a.value * b.value
        inn, hal = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
        self._rc(self._lib.swf_download_mask(self.ctx, inn.ctypes.data_as(A.PI),
                                             hal.ctypes.data_as(A.PI), C.byref(a), C.byref(b)))
        return inn[:n].reshape(b.value, a.value), hal[:n].reshape(b.value, a.value)

    # P2P halo (include/swf.h "P2P halo")
    def device_buffers(self):
        out = (C.c_void_p * 6)()
        self._rc(self._lib.swf_device_buffers(self.ctx, out))
        return [out[q] for q in range(6)]

    def set_peer(self, side: int, ptrs, peer_row0: int):
        arr = (C.c_void_p * 6)(*ptrs) if ptrs is not None else None
        self._rc(self._lib.swf_strip_set_peer(self.ctx, side, arr, int(peer_row0)))

    # asynchronous steps (include/swf.h "Asynchronous strip steps")
    def begin_batch(self):
        self._rc(self._lib.swf_strip_begin_batch(self.ctx))

    def forces(self, part: int, dt_cap: float = 0.0):
        self._rc(self._lib.swf_strip_forces(self.ctx, float(dt_cap), int(part)))

    def local_speed(self, dev_ptr: int):
        self._rc(self._lib.swf_strip_local_speed(self.ctx, C.c_void_p(dev_ptr)))

    def finish(self, dev_speed_ptr: int, dt_cap: float = 0.0):
        self._rc(self._lib.swf_strip_finish(self.ctx, C.c_void_p(dev_speed_ptr), float(dt_cap)))

    def end_batch(self):
        from ._marshal import info_from_c
        done = C.c_int()
        info = A.swf_step_info()
        self._rc(self._lib.swf_strip_end_batch(self.ctx, C.byref(done), C.byref(info)))
        return done.value, info_from_c(info)

    def steps_done(self) -> int:
        return int(self._lib.swf_strip_steps_done(self.ctx))

    def settle(self, ok: int):
        self._rc(self._lib.swf_strip_settle(self.ctx, int(ok)))

    def pack_async(self, side: int, dev_ptr: int):
        self._rc(self._lib.swf_strip_pack_async(self.ctx, side, C.c_void_p(dev_ptr)))

    def unpack_async(self, side: int, dev_ptr: int):
        self._rc(self._lib.swf_strip_unpack_async(self.ctx, side, C.c_void_p(dev_ptr)))

    def set_timing(self, slots: int):
        self._rc(self._lib.swf_set_timing(self.ctx, int(slots)))

    def timing_read(self, n: int) -> np.ndarray:
        out = np.zeros((n, 8))
        self._rc(self._lib.swf_timing_read(self.ctx, int(n), A.dptr(out)))
        return out


# ---------------------------------------------------------------------------
# exchange protocol (device-agnostic: works with NCCL on CUDA tensors and with
# gloo on CPU tensors, which is how the CPU tests exercise it)
# ---------------------------------------------------------------------------

def exchange_plan(rank: int, world: int):
    """(side, peer) pairs this rank exchanges with: side 0 = south (rank-1),
    side 1 = north (rank+1)."""
    plan = []
    if rank > 0:
        plan.append((0, rank - 1))
    if rank < world - 1:
        plan.append((1, rank + 1))
    return plan


def dist_exchange(pack, unpack, counts, rank: int, world: int, device):
    """Halo exchange through torch.distributed point-to-point ops.
    pack(side, tensor) fills a send buffer, unpack(side, tensor) consumes a
    received one; counts[side] = doubles per field."""
    import torch
    import torch.distributed as dist
    ops, recv = [], {}
    for side, peer in exchange_plan(rank, world):
        n = 3 * counts[side]
        sbuf = torch.empty(n, dtype=torch.float64, device=device)
        pack(side, sbuf)
        rbuf = torch.empty(n, dtype=torch.float64, device=device)
        ops.append(dist.P2POp(dist.isend, sbuf, peer))
        ops.append(dist.P2POp(dist.irecv, rbuf, peer))
        recv[side] = rbuf
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    if device is not None and str(device).startswith("cuda"):
        torch.cuda.synchronize(device)
    for side, rbuf in recv.items():
        unpack(side, rbuf)


def dist_allreduce_max(x: float, device) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def local_exchange(strips: Sequence[Strip]):
    """Virtual ranks on one device: strip r's south rows -> strip r-1's
    north ghosts and vice versa, through the same pack/unpack entry points."""
    import torch
    for r in range(len(strips) - 1):
        lo, hi = strips[r], strips[r + 1]
        a = torch.empty(3 * lo.count[1], dtype=torch.float64, device="cuda")
        b = torch.empty(3 * hi.count[0], dtype=torch.float64, device="cuda")
        lo.pack(1, a.data_ptr())
        hi.pack(0, b.data_ptr())
        hi.unpack(0, a.data_ptr())
        lo.unpack(1, b.data_ptr())


def local_step(strips: Sequence[Strip], dt_cap: float = 0.0):
    local_exchange(strips)
    speed = max(s.phase1(dt_cap) for s in strips)
    return [s.phase2(speed, dt_cap) for s in strips]


def local_steps_async(strips: Sequence[Strip], n: int, dt_cap: float = 0.0):
    """n steps of virtual ranks on one device through the asynchronous strip
    path (interior forces before the exchange, ghost-dependent rows after it,
    the allreduce-max on the device).  The strips' streams are ordered with
    device synchronisation here; the per-strip call sequence is exactly the
    NCCL one (RankStrip.step_async)."""
    import torch
    speeds = torch.zeros(len(strips), dtype=torch.float64, device="cuda")
    gmax = torch.zeros(1, dtype=torch.float64, device="cuda")
    bufs = {}
    for r, s in enumerate(strips):
        for side in (0, 1):
            if s.count[side]:
                bufs[(r, side)] = torch.empty(3 * s.count[side], dtype=torch.float64, device="cuda")
    for s in strips:
        s.begin_batch()
    for _ in range(n):
        for r, s in enumerate(strips):
            for side in (0, 1):
                if (r, side) in bufs:
                    s.pack_async(side, bufs[(r, side)].data_ptr())
            s.forces(0, dt_cap)
        torch.cuda.synchronize()
        for r in range(len(strips) - 1):  # the exchange: neighbour packs -> ghost rows
            strips[r + 1].unpack_async(0, bufs[(r, 1)].data_ptr())
            strips[r].unpack_async(1, bufs[(r + 1, 0)].data_ptr())
        for r, s in enumerate(strips):
            s.forces(1, dt_cap)
            s.local_speed(speeds[r:r + 1].data_ptr())
        torch.cuda.synchronize()
        # the MAX over the int64 view of the speeds (like the NCCL path)
        gmax.view(torch.int64).copy_(speeds.view(torch.int64).max().reshape(1))
        torch.cuda.synchronize()
        for s in strips:
            s.finish(gmax.data_ptr(), dt_cap)
        torch.cuda.synchronize()
    res, errs = [], []
    for s in strips:
        try:
            res.append(s.end_batch())
            errs.append(None)
        except Exception as e:  # noqa: BLE001 -- re-raised below
            res.append((s.steps_done(), None))
            errs.append(e)
    ok = min(r[0] for r in res)
    for s in strips:
        s.settle(ok)
    for e in errs:  # the first strip's own error (not a peer stop) wins
        if e is not None and "strip stopped" not in str(e):
            raise e
    for e in errs:
        if e is not None:
            raise e
    return res


# ---------------------------------------------------------------------------
# bench (torchrun, one rank per GPU)
# ---------------------------------------------------------------------------

class RankStrip:
    """One rank's strip of a scenario plus its exchange/allreduce step, over
    torch.distributed: NCCL on device buffers (production), or gloo with host
    staging (SWF_DIST_BACKEND=gloo; lets 2+ ranks share one GPU in tests)."""

    def __init__(self, config: str, n_full: int = 0, no_skip: bool = False, scenario=None):
        """config: a BASELINE.json config id, or `scenario` (a full-grid
        scenarios.Scenario, e.g. a test's random case) with config "custom"."""
        import torch
        import torch.distributed as dist
        from . import scenarios as S
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        ndev = max(1, torch.cuda.device_count())
        self.local = local % ndev
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        # NCCL needs one rank per GPU; more ranks than visible GPUs (e.g.
        # `bench.py --gpus 2` on a one-GPU box) share devices through gloo
        # with host-staged halos -- the same strip code, said on stderr
        self.backend = os.environ.get("SWF_DIST_BACKEND") or (
            "nccl" if self.world <= ndev else "gloo")
        if self.backend == "gloo" and "SWF_DIST_BACKEND" not in os.environ and self.rank == 0:
            import sys
            print(f"multigpu: {self.world} ranks on {ndev} visible GPU(s): gloo with host-staged "
                  "halos (NCCL needs one rank per GPU)", file=sys.stderr, flush=True)
        # rank 0 prints exactly one JSON line on stdout: NCCL's log goes to
        # stderr, at INFO for the communicator set-up (rank count, transports,
        # NVLS) unless the caller chose a level
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if not dist.is_initialized():
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group(self.backend)
        self.xdev = self.dev if self.backend == "nccl" else torch.device("cpu")
        self.weak = config == "C5W"
        self.full_sc = scenario
        if scenario is not None:
            self.n, self.ny = scenario.terrain.nx, scenario.terrain.ny
        else:
            self.n = n_full or {"C3": 16384, "C5": 32768, "C2": 2048, "C5W": 32768}[config]
            # rows of the global grid: square, or 4096 per GPU for weak scaling
            self.ny = S.WEAK_ROWS * self.world if self.weak else self.n
        # strips balanced by the initial activity of each block row (the wet
        # area is unevenly spread over the rows; equal row counts would leave
        # the busiest strip ~18 % above the mean at 8 GPUs on C3)
        # block size of the strips' masks (the configs use the default 16)
        self.bs = scenario.options.block_size if scenario is not None else 16
        if scenario is not None:
            self.bounds = strip_bounds(self.ny, self.world, self.bs)
        elif self.world > 1 and config in ("C3", "C5") and \
                os.environ.get("SWF_BALANCE_STRIPS", "1") != "0":
            wts = row_weights(config, self.n, 16, device=f"cuda:{self.local}")
            self.bounds = balanced_bounds(wts, self.world, 16, self.n)
        else:
            self.bounds = strip_bounds(self.ny, self.world, 16)
        self.config, self.n_full, self.no_skip = config, n_full, no_skip
        self._make_strip()
        self.strip.upload(self.sc.state.H, self.sc.state.HUx, self.sc.state.HUy, 0.0)

    def _make_strip(self):
        """The strip context of self.bounds[rank] with its window of the
        scenario (terrain, Manning field, sources, wind)."""
        from . import scenarios as S
        config, n_full, no_skip = self.config, self.n_full, self.no_skip
        self.j0, self.j1 = self.bounds[self.rank]
        self.w0, self.w1 = window_rows(self.j0, self.j1, self.ny)
        if self.full_sc is not None:
            sc = S.window_of(self.full_sc, self.w0, self.w1)
        elif self.weak:
            sc = S.build("C5", device=f"cuda:{self.local}",
                         window=(0, self.w0, self.n, self.w1 - self.w0))
        elif config in ("C3", "C5") and n_full:
            sc = S.floodplain(self.n, 50.0, window=(0, self.w0, self.n, self.w1 - self.w0),
                              device=f"cuda:{self.local}")
        else:
            sc = S.build(config, device=f"cuda:{self.local}",
                         window=(0, self.w0, self.n, self.w1 - self.w0))
        if no_skip:
            sc.options.skip_dry_blocks = False
        self.sc = sc
        import torch
        torch.cuda.empty_cache()  # the generator's device tensors, before the strip allocates
        srcs = S.clip_sources(sc.global_sources, self.n, self.ny) if self.weak else sc.global_sources
        self.strip = Strip(sc, self.ny, self.j0, self.j1, srcs, sc.wind, device=self.local)

    # ---- dynamic rebalancing ----------------------------------
    def block_row_weights(self, dry_cost: float = 0.1) -> np.ndarray:
        """This rank's owned block rows' cost in the last step: the cells of
        flux-active blocks (k_step runs them) plus dry_cost per other cell."""
        inn, hal = self.strip.mask()
        act = ((inn > 0) | (hal > 0)).sum(axis=1).astype(np.float64)
        nbx = inn.shape[1]
        return (act + dry_cost * (nbx - act)) * float(self.bs * self.bs)

    def rebalance(self, threshold: float = 0.03) -> bool:
        """Re-cut the strips from the current activity when that lowers the
        busiest strip's load by more than `threshold`; outside a batch.
        Returns whether the strips moved (every rank returns the same)."""
        import torch.distributed as dist
        if self.weak or self.world == 1:
            return False
        parts = [None] * self.world
        dist.all_gather_object(parts, self.block_row_weights())
        w = np.concatenate(parts)
        new = rebalance_bounds(w, self.bounds, self.bs, self.ny, threshold)
        if new is None:
            return False
        self.migrate(new)
        return True

    def migrate(self, new_bounds):
        """Move to new strip bounds: the rows each rank's new window needs
        travel from their current owners (transfer_plan, NCCL or gloo), the
        strip context is rebuilt for the new window and the state uploaded;
        the P2P halo, if on, is mapped again.  Same results as before the
        move, bit for bit (the state is copied, not recomputed)."""
        import torch
        import torch.distributed as dist
        new_bounds = [tuple(b) for b in new_bounds]
        old_bounds = [tuple(b) for b in self.bounds]
        nx = self.n
        H, X, Y = (np.empty((self.w1 - self.w0) * nx) for _ in range(3))
        t = self.strip.download(H, X, Y)
        own = np.stack([a.reshape(self.w1 - self.w0, nx)[self.j0 - self.w0:self.j1 - self.w0]
                        for a in (H, X, Y)])  # (3, owned rows, nx)
        nw0, nw1 = window_rows(*new_bounds[self.rank], self.ny)
        win = np.empty((3, nw1 - nw0, nx))
        ops, recvs = [], []
        for src, dst, a, b in transfer_plan(old_bounds, new_bounds, self.ny):
            if src == self.rank and dst == self.rank:
                win[:, a - nw0:b - nw0] = own[:, a - self.j0:b - self.j0]
            elif src == self.rank:
                buf = torch.from_numpy(np.ascontiguousarray(own[:, a - self.j0:b - self.j0]))
                buf = buf.to(self.xdev)
                ops.append(dist.P2POp(dist.isend, buf, dst))
                recvs.append(buf)  # keep alive until the exchange completes
            elif dst == self.rank:
                buf = torch.empty((3, b - a, nx), dtype=torch.float64, device=self.xdev)
                ops.append(dist.P2POp(dist.irecv, buf, src))
                recvs.append((buf, a, b))
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
        for r in recvs:
            if isinstance(r, tuple):
                buf, a, b = r
                win[:, a - nw0:b - nw0] = buf.cpu().numpy()
        # a fresh context for the new window
        for dp in getattr(self, "_ipc", []):
            from cuda.bindings import runtime as rt
            rt.cudaIpcCloseMemHandle(dp)
        self._ipc = []
        dist.barrier()  # every rank has unmapped its neighbours' buffers
        was_p2p = getattr(self, "p2p", False)
        self.strip.close()
        self._abufs = None
        if hasattr(self, "_tok"):
            del self._tok
        self.bounds = new_bounds
        self._make_strip()
        self.strip.upload(np.ascontiguousarray(win[0]).reshape(-1),
                          np.ascontiguousarray(win[1]).reshape(-1),
                          np.ascontiguousarray(win[2]).reshape(-1), t)
        if was_p2p:
            self.p2p = False
            self.setup_p2p()

    def _pack(self, side, t):
        import torch
        if t.is_cuda:
            self.strip.pack(side, t.data_ptr())
        else:
            tmp = torch.empty(t.numel(), dtype=torch.float64, device=self.dev)
            self.strip.pack(side, tmp.data_ptr())
            t.copy_(tmp.cpu())

    def _unpack(self, side, t):
        if t.is_cuda:
            self.strip.unpack(side, t.data_ptr())
        else:
            tmp = t.to(self.dev)
            self.strip.unpack(side, tmp.data_ptr())

    def step(self, dt_cap: float = 0.0):
        dist_exchange(self._pack, self._unpack, self.strip.count, self.rank, self.world, self.xdev)
        sp = self.strip.phase1(dt_cap)
        g = dist_allreduce_max(sp, self.xdev)
        return self.strip.phase2(g, dt_cap)

    # ---- P2P halo: k_step stores the boundary rows into the neighbours ----
    def setup_p2p(self) -> bool:
        """Map the neighbours' state buffers into this process (CUDA IPC,
        peer access over NVLink between GPUs, or the same device) and register
        them with the strip context, so the halo travels inside k_step (peer
        stores + a system fence) and a step only exchanges a 4-byte token.
        The ghost rows of the current buffer are filled once by a regular
        exchange.  Returns False (and keeps the copy exchange) when IPC is
        unavailable; every rank must agree, so the outcome is allreduced."""
        import torch
        import torch.distributed as dist
        from cuda.bindings import runtime as rt
        ok = True
        handles = None
        try:
            hs = []
            for p in self.strip.device_buffers():
                err, h = rt.cudaIpcGetMemHandle(p)
                if err != rt.cudaError_t.cudaSuccess:
                    raise RuntimeError(f"cudaIpcGetMemHandle: {err}")
                hs.append(bytes(h.reserved))
            handles = (hs, self.w0)
        except Exception:
            ok = False
        objs = [None] * self.world
        dist.all_gather_object(objs, (handles, ok))
        ok = all(o[1] for o in objs)
        opened = []
        if ok:
            try:
                for side, peer in exchange_plan(self.rank, self.world):
                    hs, peer_w0 = objs[peer][0]
                    ptrs = []
                    for hb in hs:
                        h = rt.cudaIpcMemHandle_t()
                        h.reserved = hb
                        err, dp = rt.cudaIpcOpenMemHandle(h, rt.cudaIpcMemLazyEnablePeerAccess)
                        if err != rt.cudaError_t.cudaSuccess:
                            raise RuntimeError(f"cudaIpcOpenMemHandle: {err}")
                        ptrs.append(int(dp))
                        opened.append(int(dp))
                    self.strip.set_peer(side, ptrs, peer_w0)
            except Exception:
                ok = False
        flag = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64, device=self.xdev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        ok = flag.item() == 1.0
        if not ok:
            for side in (0, 1):
                try:
                    self.strip.set_peer(side, None, 0)
                except Exception:
                    pass
            for dp in opened:
                rt.cudaIpcCloseMemHandle(dp)
            self.p2p = False
            return False
        # fill the current buffer's ghost rows once
        dist_exchange(self._pack, self._unpack, self.strip.count, self.rank, self.world, self.xdev)
        self.p2p = True
        self._ipc = opened
        return True

    def _token(self):
        """The per-step synchronisation of the P2P halo: a 1-element
        exchange with each neighbour, stream-ordered after this rank's last
        k_step (whose peer stores it publishes) and before the boundary forces."""
        import torch
        import torch.distributed as dist
        ops = []
        if not hasattr(self, "_tok"):
            self._tok = {s: (torch.zeros(1, dtype=torch.float64, device=self.xdev),
                             torch.zeros(1, dtype=torch.float64, device=self.xdev))
                         for s, _ in exchange_plan(self.rank, self.world)}
        for side, peer in exchange_plan(self.rank, self.world):
            sb, rb = self._tok[side]
            ops.append(dist.P2POp(dist.isend, sb, peer))
            ops.append(dist.P2POp(dist.irecv, rb, peer))
        return dist.batch_isend_irecv(ops) if ops else []

    def step_p2p(self, dt_cap: float = 0.0):
        """Host-synchronised P2P step (gloo tests): the neighbours' k_step
        already wrote our ghost rows; the token orders their completion."""
        import torch
        torch.cuda.synchronize(self.dev)
        for w in self._token():
            w.wait()
        sp = self.strip.phase1(dt_cap)
        g = dist_allreduce_max(sp, self.xdev)
        info = self.strip.phase2(g, dt_cap)
        return info

    # ---- NCCL, asynchronous: no host synchronisation inside a batch -------
    def _async_setup(self):
        import torch
        if getattr(self, "_abufs", None) is not None:
            return
        self._stream = torch.cuda.ExternalStream(self.strip.stream_handle(), device=self.dev)
        self._abufs = {}
        for side, peer in exchange_plan(self.rank, self.world):
            n = 3 * self.strip.count[side]
            self._abufs[side] = (torch.empty(n, dtype=torch.float64, device=self.dev),
                                 torch.empty(n, dtype=torch.float64, device=self.dev))
        self._speed = torch.zeros(1, dtype=torch.float64, device=self.dev)

    def begin_async(self):
        self._async_setup()
        self.strip.begin_batch()

    def step_async(self, dt_cap: float = 0.0):
        """One step enqueued on the strip's stream: pack, NCCL send/recv on
        the comm stream while the interior tile rows' forces run, unpack and
        the ghost-dependent rows, NCCL allreduce-MAX of the device speed,
        tau and K4..K8 from the device value."""
        import torch
        import torch.distributed as dist
        with torch.cuda.stream(self._stream):
            if getattr(self, "p2p", False):
                # the halo arrived inside the neighbours' k_step (peer stores);
                # only the ordering token crosses the links here
                works = self._token()
                self.strip.forces(0, dt_cap)  # overlaps the token
                for w in works:
                    w.wait()
                self.strip.forces(1, dt_cap)
            else:
                ops = []
                for side, peer in exchange_plan(self.rank, self.world):
                    sbuf, rbuf = self._abufs[side]
                    self.strip.pack_async(side, sbuf.data_ptr())
                    ops.append(dist.P2POp(dist.isend, sbuf, peer))
                    ops.append(dist.P2POp(dist.irecv, rbuf, peer))
                works = dist.batch_isend_irecv(ops) if ops else []
                self.strip.forces(0, dt_cap)  # overlaps the exchange
                for w in works:
                    w.wait()  # the strip stream waits for the comm stream (device side)
                for side, (sbuf, rbuf) in self._abufs.items():
                    self.strip.unpack_async(side, rbuf.data_ptr())
                self.strip.forces(1, dt_cap)
            self.strip.local_speed(self._speed.data_ptr())
            # int64 MAX over the speed bits: exact for non-negative doubles,
            # and a stopped strip's marker (swf.h) wins and stops every rank
            dist.all_reduce(self._speed.view(torch.int64), op=dist.ReduceOp.MAX)
            self.strip.finish(self._speed.data_ptr(), dt_cap)

    def end_async(self):
        """Synchronise the batch and commit the same number of steps on every
        rank: a rank that aborted in step k stopped the others in step k + 1,
        so the ranks that finished one step more roll it back
        (swf_strip_settle).  Errors are raised after the settlement."""
        import torch
        import torch.distributed as dist
        err, res = None, None
        try:
            res = self.strip.end_batch()
            done = res[0]
        except Exception as e:  # noqa: BLE001 -- re-raised below
            err, done = e, self.strip.steps_done()
        t = torch.tensor([done], dtype=torch.int64, device=self.xdev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ok = int(t.item())
        self.strip.settle(ok)
        if err is not None:
            raise err
        return (ok, res[1]) if ok == res[0] else (ok, None)

    def gather_state(self):
        """Full-grid state on rank 0 (None elsewhere)."""
        import torch
        import torch.distributed as dist
        win = self.sc.state
        H, X, Y = np.empty_like(win.H), np.empty_like(win.H), np.empty_like(win.H)
        t = self.strip.download(H, X, Y)
        r0 = (self.j0 - self.w0) * self.n
        own = np.concatenate([a[r0:r0 + (self.j1 - self.j0) * self.n] for a in (H, X, Y)])
        objs = [None] * self.world
        dist.all_gather_object(objs, (self.j0, self.j1, own, t))
        if self.rank != 0:
            return None
        n = self.n
        out = [np.empty(n * self.ny) for _ in range(3)]
        for j0, j1, o, _ in objs:
            m = (j1 - j0) * n
            for q in range(3):
                out[q][j0 * n:j1 * n] = o[q * m:(q + 1) * m]
        return out, t


def bench_strips(args) -> Optional[dict]:
    import torch
    import torch.distributed as dist
    from .scenarios import WEAK_ROWS as S_WEAK

    rs = RankStrip(args.config, no_skip=args.no_skip)
    rank, world, dev, strip, sc = rs.rank, rs.world, rs.dev, rs.strip, rs.sc
    local = rs.local
    full_n, bounds, j0, j1 = rs.n, rs.bounds, rs.j0, rs.j1
    full_ny = rs.ny
    bs = 16

    use_async = rs.backend == "nccl"
    # the halo travels inside k_step (peer stores into the neighbours' ghost
    # rows) unless SWF_HALO=copy or CUDA IPC is unavailable on this box
    p2p = use_async and os.environ.get("SWF_HALO", "p2p") != "copy" and rs.setup_p2p()

    def step():
        return rs.step(0.0)

    if use_async:  # device-side exchange/allreduce, no host sync per step
        rs.begin_async()
        for _ in range(args.warmup):
            rs.step_async(0.0)
        rs.end_async()
    else:
        for _ in range(args.warmup):
            step()
    # dynamic rebalancing from the activity after the warm-up,
    # outside the timed region; the strips keep the new cuts
    t_rb = time.perf_counter()
    rebalanced = rs.rebalance() if os.environ.get("SWF_REBALANCE", "1") != "0" else False
    t_rb = time.perf_counter() - t_rb
    if rebalanced:
        strip, sc, bounds, j0, j1 = rs.strip, rs.sc, rs.bounds, rs.j0, rs.j1
        p2p = getattr(rs, "p2p", False)
    K = args.steps
    strip.set_timing(K)
    stream = torch.cuda.ExternalStream(strip.stream_handle())
    from bench import ClockSampler, peaks, ncu_traffic  # noqa
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if use_async:
        rs.begin_async()
        e0.record(stream)
        for _ in range(K):
            rs.step_async(0.0)
        e1.record(stream)
        done, last_info = rs.end_async()
        infos = [last_info]
    else:
        e0.record(stream)
        infos = [step() for _ in range(K)]
        e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=rs.xdev)
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    clk = clocks.stop() if clocks else None
    tk = strip.timing_read(K)
    t_kstep = float(tk[:, 6].mean())
    last = infos[-1]
    N_total = full_n * full_ny
    n_own = (j1 - j0) * full_n
    n_act = min(n_own, last.flux_blocks * bs * bs) if sc.options.skip_dry_blocks else n_own
    per_act = 56 + (8 if sc.params.n_field is not None else 0)
    alg = per_act * n_act + 8 * (n_own - n_act)
    # aggregate kernel-level bandwidth: sum of per-rank algorithmic bytes / max k_step time
    nact_all = torch.tensor([float(n_act)], dtype=torch.float64, device=rs.xdev)
    dist.all_reduce(nact_all, op=dist.ReduceOp.SUM)
    agg = torch.tensor([alg, t_kstep], dtype=torch.float64, device=rs.xdev)
    alg_all = agg[0:1].clone()
    dist.all_reduce(alg_all, op=dist.ReduceOp.SUM)
    tmax = agg[1:2].clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    value = N_total * K / (ms_max * 1e-3) / 1e6

    # ---- end to end: every rank steps its strip from pinned host buffers ----
    E = max(1, getattr(args, "e2e_steps", 1))
    pin = lambda a: torch.from_numpy(np.array(a, copy=True)).pin_memory().numpy()
    hH, hX, hY = pin(sc.state.H), pin(sc.state.HUx), pin(sc.state.HUy)
    t_now = strip.download(hH, hX, hY)

    def host_step(t):
        # the strip's host-buffer step: window depth in full, momentum of the
        # flux-active owned tiles and the ghost rows over PCIe, the speeds
        # max-reduced, k_step writing the owned cells back in place
        sp = strip.host_phase1(hH, hX, hY, t)
        g = dist_allreduce_max(sp, rs.xdev)
        t, _ = strip.host_phase2(hH, hX, hY, g)
        return t

    t_now = host_step(t_now)  # warm-up of the host path
    dist.barrier()
    h2d = d2h = 0
    t0 = time.perf_counter()
    for _ in range(E):
        t_now = host_step(t_now)
        na, _, cpt = strip.active_tiles()
        h2d += strip.last_ingest_bytes() + 8
        d2h += 3 * 8 * na * cpt + 8
    el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=rs.xdev)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    io = torch.tensor([h2d / E, d2h / E], dtype=torch.float64, device=rs.xdev)
    dist.all_reduce(io, op=dist.ReduceOp.SUM)
    e2e = {"value": round(N_total * E / float(el.item()) / 1e6, 3), "unit": "Mcells/s",
           "h2d_bytes_per_step": int(io[0].item()), "d2h_bytes_per_step": int(io[1].item()),
           "how": "every rank, every step, from its pinned window of the host state "
                  "(swf_strip_host_phase1/2): depth copied in full, momentum of the "
                  "flux-active tiles and ghost rows read over PCIe, CFL speed max-reduced "
                  "across ranks, k_step writing the updated owned cells straight into the "
                  "pinned arrays; d2h counts the flux-active tiles (an upper bound); "
                  "host-timed, max over ranks"}
    if rank != 0:
        dist.barrier()
        return None
    hbm_peak, src = peaks()
    achieved = float(alg_all.item()) / float(tmax.item()) / 1e9 / world
    traffic = ncu_traffic("k_step")
    line = {
        "metric": "cell-updates/sec (Mcells/s)", "value": round(value, 3), "unit": "Mcells/s",
        "value_active": round(float(nact_all.item()) * K / (ms_max * 1e-3) / 1e6, 3),
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": round(ms_max / K, 4),
        "higher_is_better": True, "scaling": "weak" if rs.weak else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator, scenarios.py)",
        "config": {"workload": (f"C5W weak scaling: {full_n}x{full_ny} ({S_WEAK} rows per GPU) "
                                "row strips" if rs.weak else
                                f"{sc.name.split('-')[0]} {full_n}x{full_n} row strips"),
                   "cells": N_total, "strips": bounds, "halo_rows": HALO,
                   "rebalanced_after_warmup": bool(rebalanced),
                   "rebalance_s": round(t_rb, 3),
                   "parallelism": f"row strips x{world}, " + (
                       "P2P halo stored by k_step into the neighbours' ghost rows (CUDA IPC over "
                       "NVLink) + a 4-byte NCCL token per neighbour overlapped with interior "
                       "forces + device allreduce-max, no host sync" if p2p else
                       "NCCL halo send/recv overlapped with interior forces + device "
                       "allreduce-max, no host sync" if use_async else
                       "halo send/recv + allreduce-max (host-synchronised)"),
                   "l2": "inputs larger than L2"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                     "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                     "traffic": traffic["bytes_per_launch"] if traffic else None,
                     "kernel": "k_step (fused K4..K8), per GPU", "peak_source": src,
                     # per-GPU kernel behaviour, from the committed one-GPU ncu capture
                     "ncu": ({"fp64_pipe_pct": traffic["fp64_pipe_pct"],
                              "issue_active_pct": traffic["issue_active_pct"],
                              "source": traffic["source"]} if traffic else None)},
        "e2e": e2e,
        "gpu_launches": 12 * K,  # + split forces launches and the device speed for the allreduce
        "clocks": clk,
        "cpu_baseline": None,
    }
    dist.barrier()
    return line
