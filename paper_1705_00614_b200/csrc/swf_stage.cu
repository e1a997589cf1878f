// swf_stage.cu — the UNFUSED stage path: one kernel per reference stage
// (stepper.hpp:88-96), writing the same full-grid scratch arrays the
// reference's span accessors expose (stepper.hpp:102-119).  It backs the
// stage API (swf_stage / swf_download_scratch), the stage-differential parity
// tests, and step() in SWF mode 1.  Every write set is guarded by the same
// block activity as the reference (lag / flux blocks at block_size B), so
// even stale scratch values match.  Diagnostics are summed in the reference's
// block order, so StepInfo volumes are bit-identical too.
//
// The fused fast path (swf_fused.cu) uses the same per-cell arithmetic from
// swf_math.cuh and is tested bit-for-bit against this path and the oracle.
#include <cuda_runtime.h>

#include <cstdio>
#include <string>

#include "swf_internal.cuh"

namespace swf {

struct Scratch {
  double *sigma, *svx, *svy, *sigma_mid;
  unsigned char* q;
  double* fn[5];  // fx, fy, fric_x, fric_y, sigma_eff
  double* fm[5];
  double *hH, *hHUx, *hHUy, *Ht, *HVtx, *HVty, *drx, *dry, *Fh, *Fvx, *Fvy;
  FaceRec *xf, *yf;
  double* cellv;   // per-cell contribution (srcvol / deficit) for ordered sums
  double* blkv;    // per-block partials
  double* vols;    // [clamp_deficit, source_volume, boundary_outflow]
  double tau_last;
};

namespace {

constexpr int TBX = 32, TBY = 8;

struct SGeo {
  int nx, ny, bs, nbx, nby, skip;
};

__device__ __forceinline__ int blk_of(const SGeo& g, int i, int j) {
  return i / g.bs + (j / g.bs) * g.nbx;
}
__device__ __forceinline__ bool lag_cell(const SGeo& g, const unsigned char* bflag, int i, int j) {
  return !g.skip || (bflag[blk_of(g, i, j)] & 1);
}
__device__ __forceinline__ bool flux_blk(const SGeo& g, const unsigned char* bflag, int ib) {
  return !g.skip || (bflag[ib] & 2);
}

// HalfView (stepper.cpp:54-74) or StateRef (forcing.hpp:64-71) over globals.
struct GView {
  const double *Hn, *HUxn, *HUyn, *hH, *hHUx, *hHUy, *drx, *dry;
  const unsigned char* q;
  const double* b;
  double eps;
  bool half;
  __device__ bool act(size_t k) const { return Hn[k] > eps || q[k] != 0; }
  __device__ double depth(size_t k) const { return (half && act(k)) ? hH[k] : Hn[k]; }
  __device__ double momx(size_t k) const { return (half && act(k)) ? hHUx[k] : HUxn[k]; }
  __device__ double momy(size_t k) const { return (half && act(k)) ? hHUy[k] : HUyn[k]; }
  __device__ Nbr nbr(bool in, size_t k) const {
    Nbr n;
    n.in = in;
    n.depth = n.eta = n.ux = n.uy = 0.0;
    if (in) {
      n.depth = depth(k);
      n.eta = n.depth + b[k];
      if (n.depth > eps) {
        n.ux = momx(k) / n.depth;
        n.uy = momy(k) / n.depth;
      }
    }
    return n;
  }
  // cell along a face-normal line; dir 0 = x, 1 = y
  __device__ LineCell line(size_t k, int dir) const {
    LineCell c;
    c.depth = depth(k);
    c.eta = c.depth + b[k];
    c.un = 0.0;
    c.ut = 0.0;
    if (c.depth > eps) {
      double mx = momx(k) / c.depth, my = momy(k) / c.depth;
      c.un = dir == 0 ? mx : my;
      c.ut = dir == 0 ? my : mx;
    }
    c.sh = act(k) ? 0.5 * (dir == 0 ? drx[k] : dry[k]) : 0.0;
    return c;
  }
};

// ---- K1 ------------------------------------------------------------------

__global__ void k_src_fields(SGeo g, const DevSrc* src, const double* sig, int nsrc,
                             double* sigma, double* svx, double* svy, unsigned char* q) {
  int i = blockIdx.x * TBX + threadIdx.x, j = blockIdx.y * TBY + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  size_t k = (size_t)i + (size_t)j * g.nx;
  double vx = 0.0, vy = 0.0;
  double s = cell_source(src, sig, nsrc, i, j, vx, vy);
  sigma[k] = s;
  svx[k] = vx;
  svy[k] = vy;
  q[k] = (s != 0.0) ? 1 : 0;
}

__global__ void k_sigma_mid(SGeo g, const DevSrc* src, const double* sig, int nsrc,
                            double* out) {
  int i = blockIdx.x * TBX + threadIdx.x, j = blockIdx.y * TBY + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  out[(size_t)i + (size_t)j * g.nx] = cell_sigma_only(src, sig, nsrc, i, j);
}

// ---- K2 / K5 force assembly (forcing.hpp:177-237) -------------------------

__global__ void k_forces(SGeo g, GView v, PhysConst P, double n_manning, const double* nf,
                         const unsigned char* bflag, const StepScalars* sc, bool mid,
                         bool has_wind, const double* sigma, bool present, const double* svx,
                         const double* svy, double* fx, double* fy, double* frx, double* fry,
                         double* fsig) {
  int i = blockIdx.x * TBX + threadIdx.x, j = blockIdx.y * TBY + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  if (!lag_cell(g, bflag, i, j)) return;
  size_t k = (size_t)i + (size_t)j * g.nx;
  double H = v.depth(k);
  double sig = present ? sigma[k] : 0.0;
  fsig[k] = sig;
  if (H <= P.eps) {
    fx[k] = 0.0;
    fy[k] = 0.0;
    frx[k] = 0.0;
    fry[k] = 0.0;
    return;
  }
  double ux = v.momx(k) / H, uy = v.momy(k) / H;
  double eta_c = H + v.b[k];
  size_t nx = g.nx;
  Nbr W = v.nbr(i > 0, k - 1), E = v.nbr(i + 1 < g.nx, k + 1);
  Nbr S = v.nbr(j > 0, k - nx), N = v.nbr(j + 1 < g.ny, k + nx);
  double n = nf ? nf[k] : n_manning;
  double wx = mid ? sc->wind_mid[0] : sc->wind_n[0];
  double wy = mid ? sc->wind_mid[1] : sc->wind_n[1];
  ForceOut o = cell_forces(H, ux, uy, eta_c, W, E, S, N, n, P, has_wind, wx, wy, sig,
                           present ? svx[k] : 0.0, present ? svy[k] : 0.0);
  fx[k] = o.fx;
  fy[k] = o.fy;
  frx[k] = o.frx;
  fry[k] = o.fry;
}

// ---- K3 (stepper.cpp:224-267) ---------------------------------------------

__global__ void k_dt(SGeo g, PhysConst P, const double* H, const double* HUx, const double* HUy,
                     const double* fx, const double* fy, const unsigned char* bflag,
                     StepScalars* sc) {
  int i = blockIdx.x * TBX + threadIdx.x, j = blockIdx.y * TBY + threadIdx.y;
  double m = 0.0;
  if (i < g.nx && j < g.ny && lag_cell(g, bflag, i, j)) {
    size_t k = (size_t)i + (size_t)j * g.nx;
    double Hk = H[k];
    if (Hk > P.eps) {
      double ux = HUx[k] / Hk, uy = HUy[k] / Hk;
      m = cfl_speed(0.0, Hk, ux, uy, fx[k], fy[k], P.g, P.h);
    }
  }
  // max of non-negative doubles == max of their bit patterns
  unsigned long long b = dbits(m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
    b = ob > b ? ob : b;
  }
  if ((threadIdx.x & 31) == 0 && b) atomicMax(&sc->speed_bits, b);
}

// ---- K4 (stepper.cpp:269-308) ---------------------------------------------

__global__ void k_predictor(SGeo g, PhysConst P, double n_manning, const double* nf,
                            const unsigned char* bflag, double tau, const double* H,
                            const double* HUx, const double* HUy, const unsigned char* q,
                            const double* sigma, const double* fnx, const double* fny,
                            const double* fnrx, const double* fnry, double* hH, double* hHUx,
                            double* hHUy) {
  int i = blockIdx.x * TBX + threadIdx.x, j = blockIdx.y * TBY + threadIdx.y;
  if (i >= g.nx || j >= g.ny || !lag_cell(g, bflag, i, j)) return;
  size_t k = (size_t)i + (size_t)j * g.nx;
  if (!(H[k] > P.eps || q[k] != 0)) return;
  double half_tau = 0.5 * tau;
  double H12, qx, qy;
  predict_cell(H[k], HUx[k], HUy[k], sigma[k], fnx[k] - fnrx[k], fny[k] - fnry[k],
               nf ? nf[k] : n_manning, half_tau, P.eps, P.g, H12, qx, qy);
  hH[k] = H12;
  hHUx[k] = qx;
  hHUy[k] = qy;
}

// ---- K6 (stepper.cpp:335-400) ---------------------------------------------

__global__ void k_corrector(SGeo g, PhysConst P, double n_manning, const double* nf,
                            const unsigned char* bflag, double tau, bool has_src,
                            const double* H, const double* HUx, const double* HUy,
                            const unsigned char* q, const double* sigma_mid,
                            const double* fmx, const double* fmy, const double* fmrx,
                            const double* fmry, const double* hH, const double* hHUx,
                            const double* hHUy, double* Ht, double* HVtx, double* HVty,
                            double* drx, double* dry, double* cellv, StepScalars* sc) {
  int i = blockIdx.x * TBX + threadIdx.x, j = blockIdx.y * TBY + threadIdx.y;
  if (i >= g.nx || j >= g.ny || !lag_cell(g, bflag, i, j)) return;
  size_t k = (size_t)i + (size_t)j * g.nx;
  cellv[k] = 0.0;
  if (!(H[k] > P.eps || q[k] != 0)) return;
  double H12 = hH[k];
  double Htk, qx, qy, sv;
  correct_cell(H[k], HUx[k], HUy[k], has_src, sigma_mid[k], H12, fmx[k] - fmrx[k],
               fmy[k] - fmry[k], nf ? nf[k] : n_manning, tau, P.eps, P.g, Htk, qx, qy, sv);
  double ux12 = 0.0, uy12 = 0.0;
  if (H12 > P.eps) {
    ux12 = hHUx[k] / H12;
    uy12 = hHUy[k] / H12;
  }
  double dx = tau * ux12, dy = tau * uy12;
  double half_h = 0.5 * P.h;
  if (fabs(dx) >= half_h || fabs(dy) >= half_h) {
    // first offending cell (row-major) of the lowest lag block
    int ib = blk_of(g, i, j);
    unsigned long long local = (unsigned long long)((j % g.bs) * g.bs + (i % g.bs));
    unsigned long long key = (ERR_CFL << 58) | ((unsigned long long)ib << 24) | local;
    atomicMin(&sc->err_key, key);
  }
  Ht[k] = Htk;
  HVtx[k] = qx;
  HVty[k] = qy;
  drx[k] = dx;
  dry[k] = dy;
  cellv[k] = sv;
}

// ---- K7 faces (stepper.cpp:402-538, 579-618) --------------------------------

// Priority of a non-finite-face report, mirroring which write to
// blk_err_[ib] survives in the reference's serial block traversal
// (stepper.cpp:441-445, 488-492, 568-577): lowest attributed block first, and
// within it the LAST face written.  Encoded so that atomicMin picks it.
__device__ __forceinline__ unsigned long long flux_err_key(const SGeo& g,
                                                          const unsigned char* bflag, int dir,
                                                          int a, int f) {
  // dir 0: x-face iface=f on row a; dir 1: y-face jface=f on column a
  int ci = dir == 0 ? f : a, cj = dir == 0 ? a : f;
  int ib = blk_of(g, ci, cj);
  int bi = ib % g.nbx, bj = ib / g.nbx;
  int i0 = bi * g.bs, j0 = bj * g.bs;
  int rank = 2, ei0 = i0, ej0 = j0;  // executor: 0 = ib-nbx, 1 = ib-1, 2 = ib
  if (dir == 0 && f == i0 && bi > 0 && !(g.skip && !(bflag[ib - 1] & 2))) {
    rank = 1;
    ei0 = i0 - g.bs;
  }
  if (dir == 1 && f == j0 && bj > 0 && !(g.skip && !(bflag[ib - g.nbx] & 2))) {
    rank = 0;
    ej0 = j0 - g.bs;
  }
  int span = g.bs + 2;
  long long within;
  if (dir == 0) within = (long long)(a - ej0) * span + (f - ei0);
  else within = (long long)span * span + (long long)(a - ei0) * span + (f - ej0);
  long long p = (long long)rank * 2 * span * span + within;
  unsigned long long pmax = (1ull << 24) - 1;
  return (ERR_FLUX << 58) | ((unsigned long long)ib << 24) | (pmax - (unsigned long long)p);
}

__global__ void k_xfaces(SGeo g, GView v, PhysConst P, const unsigned char* bflag,
                         int west_refl, int east_refl, FaceRec* xf, StepScalars* sc) {
  int f = blockIdx.x * TBX + threadIdx.x, j = blockIdx.y * TBY + threadIdx.y;
  if (f > g.nx || j >= g.ny) return;
  // needed when a flux block touches the face
  bool need = !g.skip || (f > 0 && (bflag[blk_of(g, f - 1, j)] & 2)) ||
              (f < g.nx && (bflag[blk_of(g, f, j)] & 2));
  if (!need) return;
  size_t nx = g.nx, row = (size_t)j * nx;
  FaceRec rec;
  if (f == 0 || f == g.nx) {
    bool lo = f == 0;
    size_t k = row + (lo ? 0 : nx - 1);
    double H = v.depth(k);
    bool wet = H > P.eps;
    double un = 0.0, ut = 0.0;
    if (wet) {
      un = v.momx(k) / H;
      ut = v.momy(k) / H;
    }
    rec = boundary_face(wet, H, un, ut, lo, lo ? west_refl : east_refl, P.g);
  } else {
    size_t ka = row + f - 1, kb = row + f;
    bool has_m = f - 2 >= 0, has_p = f + 1 < g.nx;
    LineCell A = v.line(ka, 0), B = v.line(kb, 0);
    LineCell M = has_m ? v.line(ka - 1, 0) : A, Pp = has_p ? v.line(kb + 1, 0) : B;
    rec = interior_face(M, has_m, A, v.b[ka], B, v.b[kb], Pp, has_p, P.eps, P.g, P.h);
    if (!face_finite(rec)) atomicMin(&sc->err_key, flux_err_key(g, bflag, 0, j, f));
  }
  xf[(size_t)f + (size_t)j * (nx + 1)] = rec;
}

__global__ void k_yfaces(SGeo g, GView v, PhysConst P, const unsigned char* bflag,
                         int south_refl, int north_refl, FaceRec* yf, StepScalars* sc) {
  int i = blockIdx.x * TBX + threadIdx.x, f = blockIdx.y * TBY + threadIdx.y;
  if (i >= g.nx || f > g.ny) return;
  bool need = !g.skip || (f > 0 && (bflag[blk_of(g, i, f - 1)] & 2)) ||
              (f < g.ny && (bflag[blk_of(g, i, f)] & 2));
  if (!need) return;
  size_t nx = g.nx;
  FaceRec rec;
  if (f == 0 || f == g.ny) {
    bool lo = f == 0;
    size_t k = (size_t)i + (lo ? 0 : (size_t)(g.ny - 1) * nx);
    double H = v.depth(k);
    bool wet = H > P.eps;
    double un = 0.0, ut = 0.0;
    if (wet) {
      un = v.momy(k) / H;
      ut = v.momx(k) / H;
    }
    rec = boundary_face(wet, H, un, ut, lo, lo ? south_refl : north_refl, P.g);
  } else {
    size_t ka = (size_t)i + (size_t)(f - 1) * nx, kb = ka + nx;
    bool has_m = f - 2 >= 0, has_p = f + 1 < g.ny;
    LineCell A = v.line(ka, 1), B = v.line(kb, 1);
    LineCell M = has_m ? v.line(ka - nx, 1) : A, Pp = has_p ? v.line(kb + nx, 1) : B;
    rec = interior_face(M, has_m, A, v.b[ka], B, v.b[kb], Pp, has_p, P.eps, P.g, P.h);
    if (!face_finite(rec)) atomicMin(&sc->err_key, flux_err_key(g, bflag, 1, i, f));
  }
  yf[(size_t)i + (size_t)f * nx] = rec;
}

// accumulate_cell, stepper.cpp:540-566 (flux blocks)
__global__ void k_accumulate(SGeo g, GView v, PhysConst P, const unsigned char* bflag,
                             const FaceRec* xf, const FaceRec* yf, double* Fh, double* Fvx,
                             double* Fvy) {
  int i = blockIdx.x * TBX + threadIdx.x, j = blockIdx.y * TBY + threadIdx.y;
  if (i >= g.nx || j >= g.ny || !flux_blk(g, bflag, blk_of(g, i, j))) return;
  size_t nx = g.nx, k = (size_t)i + (size_t)j * nx;
  const FaceRec& W = xf[(size_t)i + (size_t)j * (nx + 1)];
  const FaceRec& E = xf[(size_t)i + 1 + (size_t)j * (nx + 1)];
  const FaceRec& S = yf[(size_t)i + (size_t)j * nx];
  const FaceRec& N = yf[(size_t)i + (size_t)(j + 1) * nx];
  double depth = v.depth(k);
  bool wet = depth > P.eps;
  double gx = 0.0, gy = 0.0;
  if (wet) {
    double eta_c = depth + v.b[k];
    Nbr Wn = v.nbr(i > 0, k - 1), En = v.nbr(i + 1 < g.nx, k + 1);
    Nbr Sn = v.nbr(j > 0, k - nx), Nn = v.nbr(j + 1 < g.ny, k + nx);
    gx = eta_grad_comp(Wn, En, eta_c, P);
    gy = eta_grad_comp(Sn, Nn, eta_c, P);
  }
  double fh, fvx, fvy;
  accumulate(W, E, S, N, wet, depth, gx, gy, P.g, P.h, fh, fvx, fvy);
  Fh[k] = fh;
  Fvx[k] = fvx;
  Fvy[k] = fvy;
}

// ---- K8 (stepper.cpp:628-674) ----------------------------------------------

__global__ void k_final(SGeo g, PhysConst P, const unsigned char* bflag, double tau, double* H,
                        double* HUx, double* HUy, const unsigned char* q, double* Ht,
                        double* HVtx, double* HVty, const double* Fh, const double* Fvx,
                        const double* Fvy, double* cellv) {
  int i = blockIdx.x * TBX + threadIdx.x, j = blockIdx.y * TBY + threadIdx.y;
  if (i >= g.nx || j >= g.ny) return;
  size_t k = (size_t)i + (size_t)j * g.nx;
  if (flux_blk(g, bflag, blk_of(g, i, j))) {
    double dt_h = tau / P.h;
    bool act = H[k] > P.eps || q[k] != 0;
    double H1, qx, qy, d;
    final_cell(act ? Ht[k] : H[k], act ? HVtx[k] : HUx[k], act ? HVty[k] : HUy[k], Fh[k],
               Fvx[k], Fvy[k], dt_h, P.eps, H1, qx, qy, d);
    H[k] = H1;
    HUx[k] = qx;
    HUy[k] = qy;
    cellv[k] = d;
  } else {
    cellv[k] = 0.0;
  }
  Ht[k] = 0.0;
  HVtx[k] = 0.0;
  HVty[k] = 0.0;
}

// Per-block partial in row-major order within the block (the reference's
// per-block serial loop), only for blocks selected by `sel` (1 lag, 2 flux).
__global__ void k_block_partials(SGeo g, const unsigned char* bflag, int sel, const double* cellv,
                                 double* blkv) {
  int ib = blockIdx.x * blockDim.x + threadIdx.x;
  if (ib >= g.nbx * g.nby) return;
  bool on = !g.skip || (bflag[ib] & sel);
  double s = 0.0;
  if (on) {
    int bi = ib % g.nbx, bj = ib / g.nbx;
    int i0 = bi * g.bs, j0 = bj * g.bs;
    int i1 = min(i0 + g.bs - 1, g.nx - 1), j1 = min(j0 + g.bs - 1, g.ny - 1);
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) s += cellv[(size_t)i + (size_t)j * g.nx];
  }
  blkv[ib] = s;
}

// Fixed-order sums (stepper.cpp:676-701), single thread: deficit over flux
// blocks, or source volume over lag blocks, in ascending block order.
__global__ void k_ordered_sum(SGeo g, const unsigned char* bflag, int sel, const double* blkv,
                              double area, double* out) {
  double s = 0.0;
  int nb = g.nbx * g.nby;
  for (int ib = 0; ib < nb; ++ib)
    if (!g.skip || (bflag[ib] & sel)) s += blkv[ib];
  *out = s * area;
}

__global__ void k_outflow(SGeo g, const unsigned char* bflag, const FaceRec* xf,
                          const FaceRec* yf, double tau, double h, double* out, StepScalars* sc) {
  double o = 0.0;
  size_t nx = g.nx;
  auto live = [&](int ci, int cj) { return !g.skip || (bflag[blk_of(g, ci, cj)] & 2); };
  for (int j = 0; j < g.ny; ++j) {
    if (live(0, j)) o -= xf[(size_t)j * (nx + 1)].fm;
    if (live(g.nx - 1, j)) o += xf[(size_t)g.nx + (size_t)j * (nx + 1)].fm;
  }
  for (int i = 0; i < g.nx; ++i) {
    if (live(i, 0)) o -= yf[i].fm;
    if (live(i, g.ny - 1)) o += yf[(size_t)i + (size_t)g.ny * nx].fm;
  }
  *out = (o * tau) * h;
  sc->t += tau;  // stepper.cpp:703
}

__global__ void k_fill(double* p, size_t n, double v) {
  size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) p[k] = v;
}

SGeo sgeo(const swf_ctx* c) {
  SGeo g;
  g.nx = c->geo.nx;
  g.ny = c->geo.ny;
  g.bs = c->geo.bs;
  g.nbx = c->geo.nbx;
  g.nby = c->geo.nby;
  g.skip = c->geo.skip;
  return g;
}

dim3 cell_grid(const SGeo& g) { return dim3((g.nx + TBX - 1) / TBX, (g.ny + TBY - 1) / TBY); }

GView view_of(swf_ctx* c, bool half) {
  Scratch* s = c->scr;
  GView v;
  v.Hn = c->H[c->cur];
  v.HUxn = c->HUx[c->cur];
  v.HUyn = c->HUy[c->cur];
  v.hH = s->hH;
  v.hHUx = s->hHUx;
  v.hHUy = s->hHUy;
  v.drx = s->drx;
  v.dry = s->dry;
  v.q = s->q;
  v.b = c->b;
  v.eps = c->geo.P.eps;
  v.half = half;
  return v;
}

int ensure_scratch(swf_ctx* c) {
  if (c->scr) return SWF_OK;
  if (c->geo.rows != c->geo.ny || c->geo.jg0 != 0)
    return set_err(c, SWF_ECONFIG, "stage API is available on whole-grid contexts only");
  Scratch* s = new Scratch();
  size_t n = local_cells(c);
  size_t nxf = (size_t)(c->geo.nx + 1) * c->geo.ny, nyf = (size_t)c->geo.nx * (c->geo.ny + 1);
  size_t nb = (size_t)c->geo.nbx * c->geo.nby;
  double** arrs[] = {&s->sigma, &s->svx, &s->svy, &s->sigma_mid, &s->fn[0], &s->fn[1],
                     &s->fn[2], &s->fn[3], &s->fn[4], &s->fm[0], &s->fm[1], &s->fm[2],
                     &s->fm[3], &s->fm[4], &s->hH, &s->hHUx, &s->hHUy, &s->Ht, &s->HVtx,
                     &s->HVty, &s->drx, &s->dry, &s->Fh, &s->Fvx, &s->Fvy, &s->cellv};
  cudaError_t e = cudaSuccess;
  for (double** a : arrs) {
    e = cudaMalloc(a, n * sizeof(double));
    if (e != cudaSuccess) break;
    cudaMemsetAsync(*a, 0, n * sizeof(double), c->stream);
  }
  if (e == cudaSuccess) e = cudaMalloc(&s->q, n);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->q, 0, n, c->stream);
  if (e == cudaSuccess) e = cudaMalloc(&s->xf, nxf * sizeof(FaceRec));
  if (e == cudaSuccess) e = cudaMemsetAsync(s->xf, 0, nxf * sizeof(FaceRec), c->stream);
  if (e == cudaSuccess) e = cudaMalloc(&s->yf, nyf * sizeof(FaceRec));
  if (e == cudaSuccess) e = cudaMemsetAsync(s->yf, 0, nyf * sizeof(FaceRec), c->stream);
  if (e == cudaSuccess) e = cudaMalloc(&s->blkv, (nb ? nb : 1) * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&s->vols, 3 * sizeof(double));
  if (e == cudaSuccess) e = cudaMemsetAsync(s->vols, 0, 3 * sizeof(double), c->stream);
  c->scr = s;
  if (e != cudaSuccess) return cuda_check(c, e, "stage scratch allocation");
  return SWF_OK;
}

int sync_and_check(swf_ctx* c) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "stage sync");
  return check_device_error(c);
}

void ev_record(swf_ctx* c, int idx) {
  if (c->timing) cudaEventRecord(c->ev[idx], c->stream);
}

}  // namespace

int stage_run(swf_ctx* c, int stage, double arg, double* tau_out) {
  int rc = ensure_scratch(c);
  if (rc) return rc;
  Scratch* s = c->scr;
  SGeo g = sgeo(c);
  dim3 grid = cell_grid(g), blk(TBX, TBY);
  const Geo& G = c->geo;
  PhysConst P = G.P;
  int H_ = c->cur;
  switch (stage) {
    case SWF_STAGE_BEGIN: {
      // begin_step, stepper.cpp:172-201: sources at t_n (only when specs
      // exist), block mask, reset diagnostics.
      rc = launch_begin(c, 0.0);
      if (rc) return rc;
      if (G.nsrc > 0)
        k_src_fields<<<grid, blk, 0, c->stream>>>(g, c->d_src, c->d_sig, G.nsrc, s->sigma, s->svx,
                                                  s->svy, s->q);
      rc = launch_mask(c);
      if (rc) return rc;
      cudaMemsetAsync(s->vols, 0, 3 * sizeof(double), c->stream);
      break;
    }
    case SWF_STAGE_FORCES: {
      GView v = view_of(c, false);
      k_forces<<<grid, blk, 0, c->stream>>>(g, v, P, G.n_manning, c->nf, c->d_bflag, c->d_sc,
                                            false, G.nwind > 0, s->sigma, G.nsrc > 0, s->svx,
                                            s->svy, s->fn[0], s->fn[1], s->fn[2], s->fn[3],
                                            s->fn[4]);
      break;
    }
    case SWF_STAGE_DT: {
      cudaMemsetAsync(&c->d_sc->speed_bits, 0, sizeof(unsigned long long), c->stream);
      k_dt<<<grid, blk, 0, c->stream>>>(g, P, c->H[H_], c->HUx[H_], c->HUy[H_], s->fn[0],
                                        s->fn[1], c->d_bflag, c->d_sc);
      // tau on the device (same kernel the fused path uses)
      rc = launch_tau(c, arg);
      if (rc) return rc;
      rc = sync_and_check(c);
      if (rc) return rc;
      if (tau_out) *tau_out = c->h_sc->tau;
      s->tau_last = c->h_sc->tau;
      break;
    }
    case SWF_STAGE_PREDICTOR: {
      k_predictor<<<grid, blk, 0, c->stream>>>(g, P, G.n_manning, c->nf, c->d_bflag, arg,
                                               c->H[H_], c->HUx[H_], c->HUy[H_], s->q, s->sigma,
                                               s->fn[0], s->fn[1], s->fn[2], s->fn[3], s->hH,
                                               s->hHUx, s->hHUy);
      break;
    }
    case SWF_STAGE_MID_FORCES: {
      // t_mid, wind(t_mid), sigma(t_mid) per spec (stepper.cpp:311-319)
      rc = launch_mid(c, arg);
      if (rc) return rc;
      if (G.nsrc > 0)
        k_sigma_mid<<<grid, blk, 0, c->stream>>>(g, c->d_src, c->d_sig + G.nsrc, G.nsrc,
                                                 s->sigma_mid);
      GView v = view_of(c, true);
      k_forces<<<grid, blk, 0, c->stream>>>(g, v, P, G.n_manning, c->nf, c->d_bflag, c->d_sc,
                                            true, G.nwind > 0, s->sigma_mid, G.nsrc > 0, s->svx,
                                            s->svy, s->fm[0], s->fm[1], s->fm[2], s->fm[3],
                                            s->fm[4]);
      break;
    }
    case SWF_STAGE_CORRECTOR: {
      k_corrector<<<grid, blk, 0, c->stream>>>(
          g, P, G.n_manning, c->nf, c->d_bflag, arg, G.nsrc > 0, c->H[H_], c->HUx[H_],
          c->HUy[H_], s->q, s->sigma_mid, s->fm[0], s->fm[1], s->fm[2], s->fm[3], s->hH,
          s->hHUx, s->hHUy, s->Ht, s->HVtx, s->HVty, s->drx, s->dry, s->cellv, c->d_sc);
      int nb = G.nbx * G.nby;
      k_block_partials<<<(nb + 127) / 128, 128, 0, c->stream>>>(g, c->d_bflag, 1, s->cellv,
                                                                  s->blkv);
      k_ordered_sum<<<1, 1, 0, c->stream>>>(g, c->d_bflag, 1, s->blkv, c->h * c->h, s->vols + 1);
      rc = sync_and_check(c);
      if (rc) return rc;
      break;
    }
    case SWF_STAGE_FLUX: {
      GView v = view_of(c, true);
      dim3 gx((g.nx + 1 + TBX - 1) / TBX, (g.ny + TBY - 1) / TBY);
      dim3 gy((g.nx + TBX - 1) / TBX, (g.ny + 1 + TBY - 1) / TBY);
      k_xfaces<<<gx, blk, 0, c->stream>>>(g, v, P, c->d_bflag, G.west_refl, G.east_refl, s->xf,
                                          c->d_sc);
      k_yfaces<<<gy, blk, 0, c->stream>>>(g, v, P, c->d_bflag, G.south_refl, G.north_refl, s->yf,
                                          c->d_sc);
      rc = sync_and_check(c);
      if (rc) return rc;
      k_accumulate<<<grid, blk, 0, c->stream>>>(g, v, P, c->d_bflag, s->xf, s->yf, s->Fh, s->Fvx,
                                                s->Fvy);
      break;
    }
    case SWF_STAGE_FINAL: {
      k_final<<<grid, blk, 0, c->stream>>>(g, P, c->d_bflag, arg, c->H[H_], c->HUx[H_],
                                           c->HUy[H_], s->q, s->Ht, s->HVtx, s->HVty, s->Fh,
                                           s->Fvx, s->Fvy, s->cellv);
      int nb = G.nbx * G.nby;
      k_block_partials<<<(nb + 127) / 128, 128, 0, c->stream>>>(g, c->d_bflag, 2, s->cellv,
                                                                  s->blkv);
      k_ordered_sum<<<1, 1, 0, c->stream>>>(g, c->d_bflag, 2, s->blkv, c->h * c->h, s->vols + 0);
      k_outflow<<<1, 1, 0, c->stream>>>(g, c->d_bflag, s->xf, s->yf, arg, c->h, s->vols + 2,
                                        c->d_sc);
      // the state changed in place: both fused buffers are stale for tiles
      if (c->d_tile_same)
        cudaMemsetAsync(c->d_tile_same, 0, (size_t)G.tiles_x * G.tiles_y, c->stream);
      invalidate_mask(c);
      break;
    }
    default:
      return set_err(c, SWF_ECONFIG, "unknown stage id");
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_check(c, e, "stage launch");
  return SWF_OK;
}

int stage_step(swf_ctx* c, double dt_cap, swf_step_info* info) {
  int rc;
  double tau = 0.0;
  float ms[8] = {0};
  cudaEvent_t* ev = c->ev;
  auto t0 = [&](int i) { ev_record(c, i); };
  t0(0);
  if ((rc = stage_run(c, SWF_STAGE_BEGIN, 0.0, nullptr))) return rc;
  t0(1);
  if ((rc = stage_run(c, SWF_STAGE_FORCES, 0.0, nullptr))) return rc;
  t0(2);
  if ((rc = stage_run(c, SWF_STAGE_DT, dt_cap, &tau))) return rc;
  t0(3);
  if ((rc = stage_run(c, SWF_STAGE_PREDICTOR, tau, nullptr))) return rc;
  t0(4);
  if ((rc = stage_run(c, SWF_STAGE_MID_FORCES, tau, nullptr))) return rc;
  t0(5);
  if ((rc = stage_run(c, SWF_STAGE_CORRECTOR, tau, nullptr))) return rc;
  t0(6);
  if ((rc = stage_run(c, SWF_STAGE_FLUX, tau, nullptr))) return rc;
  t0(7);
  if ((rc = stage_run(c, SWF_STAGE_FINAL, tau, nullptr))) return rc;
  t0(8);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "stage step");
  if (info) {
    double vols[3];
    cudaMemcpy(vols, c->scr->vols, sizeof vols, cudaMemcpyDeviceToHost);
    e = cudaMemcpy(c->h_sc, c->d_sc, sizeof(StepScalars), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_check(c, e, "stage info");
    info->tau = tau;
    fill_block_counts(c, c->h_sc, info);
    info->clamp_deficit_volume = vols[0];
    info->source_volume = vols[1];
    info->boundary_outflow_volume = vols[2];
    if (c->timing) {
      for (int i = 0; i < 8; ++i) cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]);
      for (int i = 0; i < 8; ++i) info->timings[i] = ms[i] * 1e-3;
    } else {
      for (int i = 0; i < 8; ++i) info->timings[i] = 0.0;
    }
  }
  cudaMemcpy(&c->h_t, &c->d_sc->t, sizeof(double), cudaMemcpyDeviceToHost);
  return SWF_OK;
}

int stage_download(swf_ctx* c, int which, double* out) {
  int rc = ensure_scratch(c);
  if (rc) return rc;
  Scratch* s = c->scr;
  const double* src = nullptr;
  switch (which) {
    case SWF_SCR_FN_FX: src = s->fn[0]; break;
    case SWF_SCR_FN_FY: src = s->fn[1]; break;
    case SWF_SCR_FN_FRIC_X: src = s->fn[2]; break;
    case SWF_SCR_FN_FRIC_Y: src = s->fn[3]; break;
    case SWF_SCR_FN_SIGMA: src = s->fn[4]; break;
    case SWF_SCR_FM_FX: src = s->fm[0]; break;
    case SWF_SCR_FM_FY: src = s->fm[1]; break;
    case SWF_SCR_FM_FRIC_X: src = s->fm[2]; break;
    case SWF_SCR_FM_FRIC_Y: src = s->fm[3]; break;
    case SWF_SCR_FM_SIGMA: src = s->fm[4]; break;
    case SWF_SCR_HALF_H: src = s->hH; break;
    case SWF_SCR_HALF_HUX: src = s->hHUx; break;
    case SWF_SCR_HALF_HUY: src = s->hHUy; break;
    case SWF_SCR_HT: src = s->Ht; break;
    case SWF_SCR_HVTX: src = s->HVtx; break;
    case SWF_SCR_HVTY: src = s->HVty; break;
    case SWF_SCR_DRX: src = s->drx; break;
    case SWF_SCR_DRY: src = s->dry; break;
    case SWF_SCR_FH: src = s->Fh; break;
    case SWF_SCR_FVX: src = s->Fvx; break;
    case SWF_SCR_FVY: src = s->Fvy; break;
    case SWF_SCR_SIGMA: src = s->sigma; break;
    case SWF_SCR_SRC_VX: src = s->svx; break;
    case SWF_SCR_SRC_VY: src = s->svy; break;
    default: return set_err(c, SWF_ECONFIG, "unknown scratch id");
  }
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = cudaMemcpy(out, src, local_cells(c) * sizeof(double), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? SWF_OK : cuda_check(c, e, "scratch download");
}

int stage_volumes(swf_ctx* c, double* v3) {
  if (!c->scr) {
    v3[0] = v3[1] = v3[2] = 0.0;
    return SWF_OK;
  }
  cudaError_t e = cudaMemcpy(v3, c->scr->vols, 3 * sizeof(double), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? SWF_OK : cuda_check(c, e, "volumes");
}

void stage_clear_sources(swf_ctx* c) {
  if (!c->scr) return;
  size_t n = local_cells(c);
  cudaMemsetAsync(c->scr->sigma, 0, n * sizeof(double), c->stream);
  cudaMemsetAsync(c->scr->svx, 0, n * sizeof(double), c->stream);
  cudaMemsetAsync(c->scr->svy, 0, n * sizeof(double), c->stream);
  cudaMemsetAsync(c->scr->q, 0, n, c->stream);
}

void stage_free(swf_ctx* c) {
  Scratch* s = c->scr;
  if (!s) return;
  double* arrs[] = {s->sigma, s->svx, s->svy, s->sigma_mid, s->fn[0], s->fn[1], s->fn[2],
                    s->fn[3], s->fn[4], s->fm[0], s->fm[1], s->fm[2], s->fm[3], s->fm[4],
                    s->hH, s->hHUx, s->hHUy, s->Ht, s->HVtx, s->HVty, s->drx, s->dry,
                    s->Fh, s->Fvx, s->Fvy, s->cellv, s->blkv, s->vols};
  for (double* a : arrs) cudaFree(a);
  cudaFree(s->q);
  cudaFree(s->xf);
  cudaFree(s->yf);
  delete s;
  c->scr = nullptr;
}

}  // namespace swf
