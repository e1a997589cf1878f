"""Choose the CPU-baseline sample of C3/C5 (bench.py cpu_reference): the
full grid is cut into 8 x 8 crops of n/8 squared cells; each crop's t = 0
flux-active block fraction (16-cell blocks: a wet cell inside or on the
one-cell ring, block.cpp:16-61) is computed from the seeded generator, the
crops are sorted by it and one crop is taken from the middle of each eighth
of that order (a stratified sample), so the sample's activity matches the
whole grid's.  Prints the crop origins for bench.py (developer tool).

    python tools/cpu_sample_crops.py [C3|C5] [crop]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def flux_fraction(H, bs=16, eps=1e-6):
    w = (H > eps)
    ny, nx = w.shape
    nby, nbx = ny // bs, nx // bs
    inner = w.reshape(nby, bs, nbx, bs).any(axis=(1, 3))
    # ring: a wet cell in the one-cell frame around the block (clamped)
    p = np.pad(w, 1, mode="edge")
    rows_above = p[0:ny:bs, 1:-1].reshape(nby, nbx, bs).any(axis=2)
    rows_below = p[bs + 1::bs, 1:-1].reshape(nby, nbx, bs).any(axis=2)
    cols_left = p[1:-1, 0:nx:bs].reshape(nby, bs, nbx).any(axis=1)
    cols_right = p[1:-1, bs + 1::bs].reshape(nby, bs, nbx).any(axis=1)
    corners = (p[0:ny:bs, 0:nx:bs] | p[0:ny:bs, bs + 1::bs] | p[bs + 1::bs, 0:nx:bs] |
               p[bs + 1::bs, bs + 1::bs])
    act = inner | rows_above | rows_below | cols_left | cols_right | corners
    return float(act.mean())


def main():
    from paper_1705_00614_b200 import scenarios as S
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    n = {"C3": 16384, "C5": 32768}[cfg]
    crop = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    step = n // 8
    fr = {}
    for bj in range(8):
        for bi in range(8):
            i0, j0 = bi * step + step // 2 - crop // 2, bj * step + step // 2 - crop // 2
            sc = S.build(cfg, window=(i0, j0, crop, crop))
            fr[(i0, j0)] = flux_fraction(sc.state.H.reshape(crop, crop))
            print(f"# crop {i0:6d} {j0:6d}: {fr[(i0, j0)]:.4f}", file=sys.stderr, flush=True)
    order = sorted(fr, key=lambda k: fr[k])
    pick = [order[8 * q + 4] for q in range(8)]
    mean_all = float(np.mean(list(fr.values())))
    mean_pick = float(np.mean([fr[k] for k in pick]))
    print(f"# all 64 crops: {mean_all:.4f}; stratified 8: {mean_pick:.4f}")
    print("CROPS =", [(int(a), int(b)) for a, b in pick])


if __name__ == "__main__":
    main()
