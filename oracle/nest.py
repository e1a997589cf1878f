"""TEST INFRASTRUCTURE ONLY.  CPU restatement of the two-level nesting of
SPEC.md [MODULE] nesting: prolong_boundary (:371-378),
restrict_feedback (:379-385) and coupled_step (:386-392), on top of the C
oracle stepper (pyorc.OracleStepper).

The reference ships no code for this module, so this oracle
restates the operator choices documented in
paper_1705_00614_b200/csrc/swf_nest.cu, operation for operation, in numpy
float64 (IEEE, no fused multiply-add), so the GPU path must match it bit for
bit.  Parity is pinned to the SPEC examples (tests/test_nest_oracle.py), not
to reference outputs: "parity unpinned" against the reference itself.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from paper_1705_00614_b200.types import ConfigError, FlowState, NumericalError


@dataclass
class Window:
    i0: int
    j0: int
    ni: int
    nj: int
    r: int
    ghost: int = 2
    two_way: bool = True

    @property
    def nxf(self) -> int:
        return self.r * self.ni + 2 * self.ghost

    @property
    def nyf(self) -> int:
        return self.r * self.nj + 2 * self.ghost



# substeps of one fine grid per coupled step before the coupling gives up
# (the device path's limit, csrc/swf_nest.cu); tests may lower it to check a
# non-converging case without a million Python substeps
MAX_SUBSTEPS = 1000000

def ghost_cells(w: Window):
    """(fi, fj) of the ghost band in the device's enumeration order: ghost
    bottom rows, ghost top rows, then (left gw, right gw) columns per middle row."""
    nxf, nyf, gw = w.nxf, w.nyf, w.ghost
    fi_b = np.tile(np.arange(nxf), gw)
    fj_b = np.repeat(np.arange(gw), nxf)
    fi_t = fi_b.copy()
    fj_t = np.repeat(np.arange(nyf - gw, nyf), nxf)
    cols = np.concatenate([np.arange(gw), np.arange(nxf - gw, nxf)])
    mid = np.arange(gw, nyf - gw)
    fi_m = np.tile(cols, mid.size)
    fj_m = np.repeat(mid, cols.size)
    return (np.concatenate([fi_b, fi_t, fi_m]).astype(np.int64),
            np.concatenate([fj_b, fj_t, fj_m]).astype(np.int64))


def _lerp(a, b, t):
    return a + t * (b - a)


def _coarse_coord(w0, f, gw, r):
    return (float(w0) + ((f - gw).astype(np.float64) + 0.5) / float(r)) - 0.5


def prolong(w: Window, cH, cU, cV, cb, cnx, fb, eps):
    """prolong_boundary (swf_nest.cu k_prolong): returns (3, nghost).
    Bilinear in eta, HUx, HUy when the 4 coarse cells are wet; weights
    renormalised over the wet cells when 1-3 are; dry when none is."""
    fi, fj = ghost_cells(w)
    xc = _coarse_coord(w.i0, fi, w.ghost, w.r)
    yc = _coarse_coord(w.j0, fj, w.ghost, w.r)
    ia = np.floor(xc).astype(np.int64)
    ja = np.floor(yc).astype(np.int64)
    tx = xc - ia.astype(np.float64)
    ty = yc - ja.astype(np.float64)
    k = [ia + ja * cnx]
    k += [k[0] + 1, k[0] + cnx]
    k += [k[2] + 1]
    h = [cH[q] for q in k]
    e = [cH[q] + cb[q] for q in k]
    uu = [cU[q] for q in k]
    vv = [cV[q] for q in k]
    wet = [hq > eps for hq in h]
    nwet = wet[0].astype(int) + wet[1] + wet[2] + wet[3]
    # all four wet: nested lerps
    eta4 = _lerp(_lerp(e[0], e[1], tx), _lerp(e[2], e[3], tx), ty)
    u4 = _lerp(_lerp(uu[0], uu[1], tx), _lerp(uu[2], uu[3], tx), ty)
    v4 = _lerp(_lerp(vv[0], vv[1], tx), _lerp(vv[2], vv[3], tx), ty)
    # some wet: bilinear weights renormalised over the wet cells (in order)
    sx, sy = 1.0 - tx, 1.0 - ty
    wts = [sx * sy, tx * sy, sx * ty, tx * ty]
    sw = np.zeros_like(tx)
    se, su, sv = sw.copy(), sw.copy(), sw.copy()
    for m in range(4):
        sw = np.where(wet[m], sw + wts[m], sw)
        se = np.where(wet[m], se + wts[m] * e[m], se)
        su = np.where(wet[m], su + wts[m] * uu[m], su)
        sv = np.where(wet[m], sv + wts[m] * vv[m], sv)
    with np.errstate(invalid="ignore", divide="ignore"):
        etap, up, vp = se / sw, su / sw, sv / sw
    part = (nwet > 0) & (nwet < 4)
    has = (nwet == 4) | (part & (sw > 0.0))
    eta = np.where(nwet == 4, eta4, etap)
    u = np.where(nwet == 4, u4, up)
    v = np.where(nwet == 4, v4, vp)
    bfk = fb[fi + fj * w.nxf]
    dep = eta - bfk
    H = np.where(has & (dep > 0.0), dep, 0.0)
    # a fine centre on a coarse centre: the depth form H_c + (b_c - b_f)
    node = (tx == 0.0) & (ty == 0.0)
    dep0 = h[0] + (cb[k[0]] - bfk)
    H = np.where(node, np.where(wet[0] & (dep0 > 0.0), dep0, 0.0), H)
    u = np.where(node, uu[0], u)
    v = np.where(node, vv[0], v)
    dry = ~(H > eps)
    u = np.where(dry, 0.0, u)
    v = np.where(dry, 0.0, v)
    return np.stack([H, u, v])


def apply_ghosts(w: Window, g0, g1, alpha, fine: FlowState, eps):
    """fine ghost band := lerp(g0, g1, alpha) (swf_nest.cu k_ghost_apply)."""
    fi, fj = ghost_cells(w)
    h = _lerp(g0[0], g1[0], alpha)
    u = _lerp(g0[1], g1[1], alpha)
    v = _lerp(g0[2], g1[2], alpha)
    dry = ~(h > eps)
    u = np.where(dry, 0.0, u)
    v = np.where(dry, 0.0, v)
    k = fi + fj * w.nxf
    fine.H[k] = h
    fine.HUx[k] = u
    fine.HUy[k] = v


def restrict(w: Window, fine: FlowState, coarse: FlowState, cnx: int):
    """restrict_feedback (swf_nest.cu k_restrict): row-major sums / r^2."""
    r, gw, nxf = w.r, w.ghost, w.nxf
    out = []
    for a in (fine.H, fine.HUx, fine.HUy):
        A = a.reshape(w.nyf, nxf)[gw:gw + r * w.nj, gw:gw + r * w.ni]
        blk = A.reshape(w.nj, r, w.ni, r)  # (cj, b, ci, a)
        s = np.zeros((w.nj, w.ni))
        for b in range(r):
            for aa in range(r):
                s = s + blk[:, b, :, aa]
        out.append(s / float(r * r))
    ny_c = coarse.H.size // cnx
    for dst, m in zip((coarse.H, coarse.HUx, coarse.HUy), out):
        D = dst.reshape(ny_c, cnx)
        D[w.j0:w.j0 + w.nj, w.i0:w.i0 + w.ni] = m


def face_taps(stepper, nx, ny, rect):
    """fm through the faces on the boundary of the cell rectangle rect =
    (i0, j0, ni, nj) after the stepper's last step, as swf_fused.cu's face
    taps record them: [west nj | east nj | south ni | north ni]; faces whose
    adjacent blocks were both inactive (not computed, dry) are 0."""
    i0, j0, ni, nj = rect
    fx = stepper.face_fm(0).reshape(ny, nx + 1)
    fy = stepper.face_fm(1).reshape(ny + 1, nx)
    jr = np.arange(j0, j0 + nj)
    ir = np.arange(i0, i0 + ni)
    w, e = fx[jr, i0].copy(), fx[jr, i0 + ni].copy()
    so, no = fy[j0, ir].copy(), fy[j0 + nj, ir].copy()
    if stepper._options.skip_dry_blocks:
        m = stepper.mask()
        bs = m.block_size
        act = ((m.interior_wet > 0) | (m.halo_wet > 0)).reshape(m.nby, m.nbx)
        fb = lambda ii, jj: act[jj // bs, ii // bs]
        w = np.where(fb(np.full_like(jr, i0 - 1), jr) | fb(np.full_like(jr, i0), jr), w, 0.0)
        e = np.where(fb(np.full_like(jr, i0 + ni - 1), jr) | fb(np.full_like(jr, i0 + ni), jr), e, 0.0)
        so = np.where(fb(ir, np.full_like(ir, j0 - 1)) | fb(ir, np.full_like(ir, j0)), so, 0.0)
        no = np.where(fb(ir, np.full_like(ir, j0 + nj - 1)) | fb(ir, np.full_like(ir, j0 + nj)), no, 0.0)
    return np.concatenate([w, e, so, no])


def reflux(w: Window, tc, tf, hc, hf, coarse: FlowState, eps):
    """swf_nest.cu k_reflux: the coarse cells outside the window trade the
    coarse step's face volumes for the fine substeps' ones."""
    nx = coarse.nx
    r, ni, nj, i0, j0 = w.r, w.ni, w.nj, w.i0, w.j0
    clamp = 0.0
    for q in range(2 * (ni + nj)):
        if q < nj:
            side, k, fo, i, j = 0, q, q * r, i0 - 1, j0 + q
        elif q < 2 * nj:
            k = q - nj
            side, fo, i, j = 1, r * nj + k * r, i0 + ni, j0 + k
        elif q < 2 * nj + ni:
            k = q - 2 * nj
            side, fo, i, j = 2, 2 * r * nj + k * r, i0 + k, j0 - 1
        else:
            k = q - 2 * nj - ni
            side, fo, i, j = 3, 2 * r * nj + r * ni + k * r, i0 + k, j0 + nj
        vc = float(tc[q]) * hc
        vf = 0.0
        for b in range(r):
            vf = vf + float(tf[fo + b])
        vf = vf * hf
        d = (vc - vf) / (hc * hc) if side in (0, 2) else (vf - vc) / (hc * hc)
        c = i + j * nx
        h = coarse.H[c] + d
        clamp = clamp + ((0.0 - h) * (hc * hc) if h < 0.0 else 0.0)
        if not (h > 0.0):
            h = 0.0
        coarse.H[c] = h
        if not (h > eps):
            coarse.HUx[c] = 0.0
            coarse.HUy[c] = 0.0
    return clamp


class OracleNest:
    """One window: its fine OracleStepper and fine FlowState."""

    def __init__(self, window: Window, fine_stepper, fine_state: FlowState, fine_b, eps):
        self.w = window
        self.fine = fine_stepper
        self.state = fine_state
        self.fb = fine_b
        self.eps = eps


def coupled_step(coarse_stepper, coarse_state: FlowState, coarse_b, nests: List[OracleNest],
                 dt_cap: float = 0.0):
    """coupled_step as swf_nest.cu swf_coupled_step does it,
    with the flux correction of two-way windows.  Returns (coarse StepInfo,
    substeps per nest); the reflux clamp volume is in coupled_step.clamp."""
    cnx = coarse_state.nx
    t0 = coarse_state.t
    coupled_step.clamp = 0.0
    g0 = []
    for n in nests:
        if n.state.t != t0:
            raise ConfigError("coupled_step: nested grid not synchronized with the global grid")
        g0.append(prolong(n.w, coarse_state.H, coarse_state.HUx, coarse_state.HUy, coarse_b, cnx,
                          n.fb, n.eps))
    info = coarse_stepper.step(coarse_state, dt_cap)
    t1 = coarse_state.t
    tau_g = t1 - t0
    hc = coarse_stepper._terrain.h
    tcs = [info.tau * face_taps(coarse_stepper, cnx, coarse_state.ny, (n.w.i0, n.w.j0, n.w.ni, n.w.nj))
           if n.w.two_way else None for n in nests]
    subs = []
    for q, n in enumerate(nests):
        g1 = prolong(n.w, coarse_state.H, coarse_state.HUx, coarse_state.HUy, coarse_b, cnx, n.fb,
                     n.eps)
        tf = t0
        tol = max(1e-9 * tau_g, 8.0 * 2.220446049250313e-16 * abs(t1))
        sub = 0
        frect = (n.w.ghost, n.w.ghost, n.w.r * n.w.ni, n.w.r * n.w.nj)
        tfs = np.zeros(2 * (frect[2] + frect[3]))
        while t1 - tf > tol:
            alpha = (tf - t0) / (t1 - t0)
            apply_ghosts(n.w, g0[q], g1, alpha, n.state, n.eps)
            fi = n.fine.step(n.state, info.tau if sub == 0 else t1 - tf)
            if n.w.two_way:
                tfs = tfs + fi.tau * face_taps(n.fine, n.w.nxf, n.w.nyf, frect)
            tf = n.state.t
            sub += 1
            if sub > MAX_SUBSTEPS:
                raise NumericalError("nested grid: subcycling does not converge")
        n.state.t = t1
        subs.append(sub)
        if n.w.two_way:
            restrict(n.w, n.state, coarse_state, cnx)
            coupled_step.clamp += reflux(n.w, tcs[q], tfs, hc, n.fine._terrain.h, coarse_state,
                                         n.eps)
    return info, subs
