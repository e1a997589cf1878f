// swf_fused.cu — the FUSED fast path of one CSPH-TVD step on sm_100a.
//
// One step = 6 launches on the context's stream (captured in a CUDA graph
// for swf_run):
//   k_begin   1 thread   sources sigma_s(t_n), wind(t_n), counter reset
//   k_mask    B-blocks   K1: interior / halo-ring activity counts (block.cpp:16-61)
//   k_tiles   tiles      fused-tile activity from the B-block flags
//   k_forces  tiles      K2 + K3: forces on wet cells (stores f - f_fric only)
//                        and the CFL speed (shuffle + one atomicMax per CTA)
//   k_tau     1 thread   tau = min(dt_max, K h / speed, dt_cap); t_mid,
//                        wind(t_mid), sigma_s(t_mid)  (stepper.cpp:256-266, 311-319)
//   k_step    tiles      K4..K8 fused: predictor on the tile + 2-cell halo,
//                        mid forces + corrector on owned cells, x- then y-face
//                        TVD/HLL fluxes in shared memory, accumulate, final
//                        update into the other state buffer (ping-pong)
//   k_finish  1 CTA      fixed-order diagnostics, t += tau
//
// HBM traffic per wet cell-update: k_forces reads H,HUx,HUy,b (+n) and writes
// 2 doubles; k_step reads H,HUx,HUy,b,f' (+n) and writes H,HUx,HUy — ≈120 B
// against the 56 B compulsory minimum; the FP64 pipe, not HBM, bounds this
// path.  Dry tiles cost one read of H in k_forces and, once
// after they go dry, one copy between the ping-pong buffers.
#include <cuda_runtime.h>

#include "swf_internal.cuh"

namespace swf {
namespace {

// ---- tiles -----------------------------------------------------------------
constexpr int AX = 32, AY = 16;  // k_forces tile (owned cells)
constexpr int AREGX = AX + 2, AREGY = AY + 2, AREG = AREGX * AREGY;
constexpr int BX = 32, BY = 16;  // k_step tile (owned cells)
constexpr int RX = BX + 4, RY = BY + 4, RREG = RX * RY;  // 2-cell halo region
constexpr int NTHR = 256;

__device__ __forceinline__ bool stopped(const StepScalars* sc) { return sc->err_key != ERR_NONE; }

// ---------------------------------------------------------------------------
// k_begin: per-step scalars at t_n (begin_step stepper.cpp:176-183,
// source_terms sources.cpp:45-64, WindForcing::at grid.cpp:64-75)
// ---------------------------------------------------------------------------
__global__ void k_begin(Geo G, const DevSrc* src, const double* ht, const double* hq,
                        const double* wt, const double* wv, double* sig, StepScalars* sc,
                        double dt_cap) {
  if (stopped(sc)) return;
  double t = sc->t;
  for (int m = 0; m < G.nsrc; ++m) {
    const DevSrc& d = src[m];
    double s;
    if (d.kind == SWF_SOURCE_RAIN) s = d.rate;
    else s = series_at(ht + d.off, hq + d.off, d.nh, 1, 0, t) / d.count_area;
    sig[m] = s;
  }
  sc->wind_n[0] = series_at(wt, wv, G.nwind, 2, 0, t);
  sc->wind_n[1] = series_at(wt, wv, G.nwind, 2, 1, t);
  sc->speed_bits = 0ull;
  sc->lag_act = 0;
  sc->flux_act = 0;
  sc->dt_cap = dt_cap;
}

// mid-step scalars for a given tau (stepper.cpp:311-319)
__device__ void mid_scalars(const Geo& G, const DevSrc* src, const double* ht, const double* hq,
                            const double* wt, const double* wv, double* sig, StepScalars* sc,
                            double tau) {
  double t_mid = sc->t + 0.5 * tau;
  sc->t_mid = t_mid;
  for (int m = 0; m < G.nsrc; ++m) {
    const DevSrc& d = src[m];
    double s;
    if (d.kind == SWF_SOURCE_RAIN) s = d.rate;
    else s = series_at(ht + d.off, hq + d.off, d.nh, 1, 0, t_mid) / d.count_area;
    sig[G.nsrc + m] = s;
  }
  sc->wind_mid[0] = series_at(wt, wv, G.nwind, 2, 0, t_mid);
  sc->wind_mid[1] = series_at(wt, wv, G.nwind, 2, 1, t_mid);
}

// k_tau: compute_dt's scalar tail (stepper.cpp:253-266) + mid scalars.
// global_speed >= 0 overrides the device max (multi-strip allreduce result).
__global__ void k_tau(Geo G, const DevSrc* src, const double* ht, const double* hq,
                      const double* wt, const double* wv, double* sig, StepScalars* sc,
                      double dt_cap, double global_speed) {
  if (stopped(sc)) return;
  double speed = global_speed >= 0.0 ? global_speed : bitsd(sc->speed_bits);
  double tau = G.dt_max;
  if (speed > 0.0) {
    double cfl = (G.courant * G.P.h) / speed;
    if (cfl < G.dt_min) {
      sc->err_val[0] = cfl;
      sc->err_val[1] = G.dt_min;
      sc->err_val[2] = speed;
      atomicMin(&sc->err_key, ERR_DT << 58);
      return;
    }
    tau = smin(tau, cfl);
  }
  if (dt_cap > 0.0) tau = smin(tau, dt_cap);
  sc->tau = tau;
  mid_scalars(G, src, ht, hq, wt, wv, sig, sc, tau);
}

__global__ void k_mid(Geo G, const DevSrc* src, const double* ht, const double* hq,
                      const double* wt, const double* wv, double* sig, StepScalars* sc,
                      double tau) {
  mid_scalars(G, src, ht, hq, wt, wv, sig, sc, tau);
}

// ---------------------------------------------------------------------------
// k_mask: K1 (compute_block_mask, block.cpp:16-61).  One thread per owned
// B-block: interior count and the clamped one-cell ring (corners included).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool wet_at(const Geo& G, const double* H, const DevSrc* src,
                                       const double* sig, int i, int jg) {
  size_t k = (size_t)i + (size_t)(jg - G.jg0) * G.nx;
  if (H[k] > G.P.eps) return true;
  return G.nsrc > 0 && cell_sigma_only(src, sig, G.nsrc, i, jg) != 0.0;
}

__global__ void k_mask(Geo G, const double* H, const DevSrc* src, const double* sig,
                       int* interior, int* halo, unsigned char* bflag, StepScalars* sc) {
  int nbl = G.nbx * (G.bj1 - G.bj0);
  int lb = blockIdx.x * blockDim.x + threadIdx.x;
  bool lag = false, flx = false;
  if (lb < nbl) {
    int bi = lb % G.nbx, bj = G.bj0 + lb / G.nbx;
    int i0 = bi * G.bs, j0 = bj * G.bs;
    int i1 = min(i0 + G.bs - 1, G.nx - 1), j1 = min(j0 + G.bs - 1, G.ny - 1);
    int in = 0, ring = 0;
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) in += wet_at(G, H, src, sig, i, j);
    int jlo = max(j0 - 1, 0), jhi = min(j1 + 1, G.ny - 1);
    for (int i = i0 - 1; i <= i1 + 1; ++i) {
      int ci = min(max(i, 0), G.nx - 1);
      ring += wet_at(G, H, src, sig, ci, jlo);
      ring += wet_at(G, H, src, sig, ci, jhi);
    }
    int ilo = max(i0 - 1, 0), ihi = min(i1 + 1, G.nx - 1);
    for (int j = j0; j <= j1; ++j) {
      ring += wet_at(G, H, src, sig, ilo, j);
      ring += wet_at(G, H, src, sig, ihi, j);
    }
    interior[lb] = in;
    halo[lb] = ring;
    lag = in > 0;
    flx = lag || ring > 0;
    bflag[lb] = (lag ? 1 : 0) | (flx ? 2 : 0);
  }
  int nl = __syncthreads_count(lag), nf = __syncthreads_count(flx);
  if (threadIdx.x == 0) {
    if (nl) atomicAdd(&sc->lag_act, nl);
    if (nf) atomicAdd(&sc->flux_act, nf);
  }
}

// k_tiles: fused-tile flags from the B-block flags.  bit0: some overlapping
// block is Lagrangian-active; bit1: some overlapping block is flux-active.
__global__ void k_tiles(Geo G, const unsigned char* bflag, unsigned char* tile_act) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= G.tiles_x * G.tiles_y) return;
  int tx = t % G.tiles_x, ty = t / G.tiles_x;
  int i0 = tx * BX, i1 = min(i0 + BX, G.nx) - 1;
  int jg0 = G.jg0 + G.r0 + ty * BY, jg1 = min(G.jg0 + G.r0 + ty * BY + BY, G.jg0 + G.r1) - 1;
  unsigned char f = 0;
  for (int bj = jg0 / G.bs; bj <= jg1 / G.bs; ++bj)
    for (int bi = i0 / G.bs; bi <= i1 / G.bs; ++bi) f |= bflag[bi + (bj - G.bj0) * G.nbx];
  if (!G.skip) f |= 3;
  tile_act[t] = f;
}

// ---------------------------------------------------------------------------
// k_forces: K2 + K3.  Tile AX x AY owned cells + 1-cell halo in shared memory.
// Writes f' = (fx - fric_x, fy - fric_y) for wet cells (the only K2 output
// the predictor needs, stepper.cpp:283-284) and reduces the CFL speed of
// K3 (stepper.cpp:233-254) with warp shuffles and one atomicMax per CTA.
// Rows [ra0, ra1) (local): owned rows plus, for strips, 2 ghost rows each
// side so k_step can run its predictor on its 2-cell halo.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NTHR) k_forces(Geo G, int ra0, int ra1, int tiles_xa,
                                                 const double* __restrict__ H,
                                                 const double* __restrict__ HUx,
                                                 const double* __restrict__ HUy,
                                                 const double* __restrict__ b,
                                                 const double* __restrict__ nf,
                                                 const DevSrc* src, const double* sig,
                                                 double* __restrict__ fpx,
                                                 double* __restrict__ fpy, StepScalars* sc) {
  __shared__ double s_d[AREG], s_e[AREG], s_u[AREG], s_v[AREG];
  if (stopped(sc)) return;
  const PhysConst& P = G.P;
  int tx = blockIdx.x % tiles_xa, ty = blockIdx.x / tiles_xa;
  int i0 = tx * AX, rr0 = ra0 + ty * AY;
  int tid = threadIdx.x;
  // activity: any wet owned cell in the tile?
  bool anywet = false;
  for (int c = tid; c < AX * AY; c += NTHR) {
    int i = i0 + c % AX, r = rr0 + c / AX;
    if (i < G.nx && r < ra1) anywet |= H[(size_t)i + (size_t)r * G.nx] > P.eps;
  }
  if (!__syncthreads_or(anywet)) return;
  for (int c = tid; c < AREG; c += NTHR) {
    int i = i0 - 1 + c % AREGX, r = rr0 - 1 + c / AREGX;
    double d = 0.0, e = 0.0, u = 0.0, v = 0.0;
    if (i >= 0 && i < G.nx && r >= 0 && r < G.rows) {
      size_t k = (size_t)i + (size_t)r * G.nx;
      d = H[k];
      e = d + b[k];
      if (d > P.eps) {
        u = HUx[k] / d;
        v = HUy[k] / d;
      }
    }
    s_d[c] = d;
    s_e[c] = e;
    s_u[c] = u;
    s_v[c] = v;
  }
  __syncthreads();
  double m = 0.0;
  double wx = sc->wind_n[0], wy = sc->wind_n[1];
  const double* sig_n = sig;
  for (int c = tid; c < AX * AY; c += NTHR) {
    int x = c % AX, y = c / AX;
    int i = i0 + x, r = rr0 + y;
    if (i >= G.nx || r >= ra1) continue;
    int s = (x + 1) + (y + 1) * AREGX;
    double d = s_d[s];
    if (!(d > P.eps)) continue;
    int jg = G.jg0 + r;
    auto nb = [&](bool in, int q) {
      Nbr n;
      n.in = in;
      n.depth = s_d[q];
      n.eta = s_e[q];
      n.ux = s_u[q];
      n.uy = s_v[q];
      return n;
    };
    Nbr W = nb(i > 0, s - 1), E = nb(i + 1 < G.nx, s + 1);
    Nbr S = nb(jg > 0, s - AREGX), N = nb(jg + 1 < G.ny, s + AREGX);
    double sg = 0.0, svx = 0.0, svy = 0.0;
    if (G.nsrc > 0) sg = cell_source(src, sig_n, G.nsrc, i, jg, svx, svy);
    size_t k = (size_t)i + (size_t)r * G.nx;
    double n = G.has_nfield ? nf[k] : G.n_manning;
    double ux = s_u[s], uy = s_v[s];
    ForceOut o = cell_forces(d, ux, uy, s_e[s], W, E, S, N, n, P, G.nwind > 0, wx, wy, sg, svx,
                             svy);
    fpx[k] = o.fx - o.frx;
    fpy[k] = o.fy - o.fry;
    m = cfl_speed(m, d, ux, uy, o.fx, o.fy, P.g, P.h);
  }
  unsigned long long bits = dbits(m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long ob = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = ob > bits ? ob : bits;
  }
  __shared__ unsigned long long s_max[NTHR / 32];
  if ((tid & 31) == 0) s_max[tid >> 5] = bits;
  __syncthreads();
  if (tid == 0) {
    unsigned long long mb = 0;
    for (int w = 0; w < NTHR / 32; ++w) mb = s_max[w] > mb ? s_max[w] : mb;
    if (mb) atomicMax(&sc->speed_bits, mb);
  }
}

// ---------------------------------------------------------------------------
// k_step: K4..K8 fused over a BX x BY tile.
// ---------------------------------------------------------------------------

// shared-memory layout of the 2-cell-halo region (RX x RY), half-step view
enum { F_D = 0, F_E, F_U, F_V, F_SX, F_SY, F_B, F_HN, F_QX, F_QY, F_NUM };

struct StepArgs {
  const double* __restrict__ H;
  const double* __restrict__ HUx;
  const double* __restrict__ HUy;
  const double* __restrict__ b;
  const double* __restrict__ nf;
  const double* __restrict__ fpx;
  const double* __restrict__ fpy;
  double* __restrict__ Ho;
  double* __restrict__ HUxo;
  double* __restrict__ HUyo;
  const DevSrc* src;
  const double* sig;  // [0,nsrc): t_n, [nsrc,2nsrc): t_mid
  const unsigned char* bflag;
  const unsigned char* tile_act;
  unsigned char* tile_same;
  double* part;  // 3 per tile
  StepScalars* sc;
};

__device__ __forceinline__ unsigned long long fused_flux_key(const Geo& G,
                                                            const unsigned char* bflag, int dir,
                                                            int a, int f) {
  // same priority as the stage path (swf_stage.cu flux_err_key), global ids
  int ci = dir == 0 ? f : a, cj = dir == 0 ? a : f;
  int bi = ci / G.bs, bj = cj / G.bs;
  int ib = bi + bj * G.nbx;
  int i0 = bi * G.bs, j0 = bj * G.bs;
  auto flx = [&](int bi2, int bj2) {
    if (bj2 < G.bj0 || bj2 >= G.bj1) return true;
    return (bflag[bi2 + (bj2 - G.bj0) * G.nbx] & 2) != 0;
  };
  int rank = 2, ei0 = i0, ej0 = j0;
  if (dir == 0 && f == i0 && bi > 0 && !(G.skip && !flx(bi - 1, bj))) {
    rank = 1;
    ei0 = i0 - G.bs;
  }
  if (dir == 1 && f == j0 && bj > 0 && !(G.skip && !flx(bi, bj - 1))) {
    rank = 0;
    ej0 = j0 - G.bs;
  }
  int span = G.bs + 2;
  long long within;
  if (dir == 0) within = (long long)(a - ej0) * span + (f - ei0);
  else within = (long long)span * span + (long long)(a - ei0) * span + (f - ej0);
  long long p = (long long)rank * 2 * span * span + within;
  unsigned long long pmax = (1ull << 24) - 1;
  return (ERR_FLUX << 58) | ((unsigned long long)ib << 24) | (pmax - (unsigned long long)p);
}

__global__ void __launch_bounds__(NTHR, 2) k_step(Geo G, StepArgs A) {
  extern __shared__ double smem[];
  double* R = smem;                  // F_NUM x RREG
  double* FB = smem + F_NUM * RREG;  // face buffer: 4 x 544
  constexpr int NF = (BX + 1) * BY > BX * (BY + 1) ? (BX + 1) * BY : BX * (BY + 1);
  const PhysConst& P = G.P;
  StepScalars* sc = A.sc;
  if (stopped(sc)) return;
  const int tid = threadIdx.x;
  const int tile = blockIdx.x;
  const int tx = tile % G.tiles_x, ty = tile / G.tiles_x;
  const int i0 = tx * BX;        // first owned column
  const int r0 = G.r0 + ty * BY; // first owned local row
  const size_t nx = G.nx;

  // ---- inactive tile: keep the step-start state (skip semantics) ----------
  if (!(A.tile_act[tile] & 2)) {
    if (!A.tile_same[tile]) {
      for (int c = tid; c < BX * BY; c += NTHR) {
        int i = i0 + c % BX, r = r0 + c / BX;
        if (i < G.nx && r < G.r1) {
          size_t k = (size_t)i + (size_t)r * nx;
          A.Ho[k] = A.H[k];
          A.HUxo[k] = A.HUx[k];
          A.HUyo[k] = A.HUy[k];
        }
      }
      if (tid == 0) A.tile_same[tile] = 1;
    }
    if (tid == 0) {
      A.part[3 * tile + 0] = 0.0;
      A.part[3 * tile + 1] = 0.0;
      A.part[3 * tile + 2] = 0.0;
    }
    return;
  }

  const double tau = sc->tau;
  const double half_tau = 0.5 * tau;
  const int nsrc = G.nsrc;
  const double* sig_n = A.sig;
  const double* sig_m = A.sig + nsrc;

  // ---- phase 1: half-step view on the region (K4 predictor, HalfView) ------
  for (int c = tid; c < RREG; c += NTHR) {
    int i = i0 - 2 + c % RX, r = r0 - 2 + c / RX;
    double d = 0.0, e = 0.0, u = 0.0, v = 0.0, sx = 0.0, sy = 0.0, bb = 0.0;
    double Hn = 0.0, qxn = 0.0, qyn = 0.0;
    if (i >= 0 && i < G.nx && r >= 0 && r < G.rows) {
      size_t k = (size_t)i + (size_t)r * nx;
      Hn = A.H[k];
      qxn = A.HUx[k];
      qyn = A.HUy[k];
      bb = A.b[k];
      double sg = 0.0;
      if (nsrc > 0) sg = cell_sigma_only(A.src, sig_n, nsrc, i, G.jg0 + r);
      bool act = Hn > P.eps || sg != 0.0;
      d = Hn;
      double mx = qxn, my = qyn;
      if (act) {
        bool wet = Hn > P.eps;
        double fx = wet ? A.fpx[k] : 0.0, fy = wet ? A.fpy[k] : 0.0;
        double n = G.has_nfield ? A.nf[k] : G.n_manning;
        predict_cell(Hn, qxn, qyn, sg, fx, fy, n, half_tau, P.eps, P.g, d, mx, my);
      }
      e = d + bb;
      if (d > P.eps) {
        u = mx / d;
        v = my / d;
      }
      if (act) {
        // shift = 0.5*dr with dr = tau * u12 (stepper.cpp:72-73, 373-379);
        // u12 equals the half view velocity for active cells
        sx = 0.5 * (tau * u);
        sy = 0.5 * (tau * v);
      }
    }
    R[F_D * RREG + c] = d;
    R[F_E * RREG + c] = e;
    R[F_U * RREG + c] = u;
    R[F_V * RREG + c] = v;
    R[F_SX * RREG + c] = sx;
    R[F_SY * RREG + c] = sy;
    R[F_B * RREG + c] = bb;
    R[F_HN * RREG + c] = Hn;
    R[F_QX * RREG + c] = qxn;
    R[F_QY * RREG + c] = qyn;
  }
  __syncthreads();

  // ---- phase 2: K5 mid forces + K6 corrector on owned active cells ---------
  constexpr int PER = BX * BY / NTHR;  // owned cells per thread (2)
  double Ht[PER], Qx[PER], Qy[PER];
  double srcvol = 0.0;
  const double wmx = sc->wind_mid[0], wmy = sc->wind_mid[1];
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    int c = tid + m * NTHR;
    int x = c % BX, y = c / BX;
    int i = i0 + x, r = r0 + y;
    Ht[m] = 0.0;
    Qx[m] = 0.0;
    Qy[m] = 0.0;
    if (i >= G.nx || r >= G.r1) continue;
    int s = (x + 2) + (y + 2) * RX;
    int jg = G.jg0 + r;
    double Hn = R[F_HN * RREG + s];
    double sgn_ = 0.0, svx = 0.0, svy = 0.0, sgm = 0.0;
    if (nsrc > 0) {
      sgn_ = cell_source(A.src, sig_n, nsrc, i, jg, svx, svy);
      sgm = cell_sigma_only(A.src, sig_m, nsrc, i, jg);
    }
    bool act = Hn > P.eps || sgn_ != 0.0;
    if (!act) continue;
    size_t k = (size_t)i + (size_t)r * nx;
    double n = G.has_nfield ? A.nf[k] : G.n_manning;
    double d = R[F_D * RREG + s];  // H12
    double fmx = 0.0, fmy = 0.0;
    if (d > P.eps) {
      auto nb = [&](bool in, int q) {
        Nbr o;
        o.in = in;
        o.depth = R[F_D * RREG + q];
        o.eta = R[F_E * RREG + q];
        o.ux = R[F_U * RREG + q];
        o.uy = R[F_V * RREG + q];
        return o;
      };
      Nbr W = nb(i > 0, s - 1), E = nb(i + 1 < G.nx, s + 1);
      Nbr S = nb(jg > 0, s - RX), N = nb(jg + 1 < G.ny, s + RX);
      ForceOut o = cell_forces(d, R[F_U * RREG + s], R[F_V * RREG + s], R[F_E * RREG + s], W,
                               E, S, N, n, P, G.nwind > 0, wmx, wmy, nsrc > 0 ? sgm : 0.0, svx,
                               svy);
      fmx = o.fx - o.frx;
      fmy = o.fy - o.fry;
    }
    double ht, qx, qy, sv;
    correct_cell(Hn, R[F_QX * RREG + s], R[F_QY * RREG + s], nsrc > 0, sgm, d, fmx, fmy, n, tau,
                 P.eps, P.g, ht, qx, qy, sv);
    srcvol += sv;
    // CFL abort (stepper.cpp:378-380, 391-399): dr = tau * u12
    double dx = tau * R[F_U * RREG + s], dy = tau * R[F_V * RREG + s];
    double half_h = 0.5 * P.h;
    if (fabs(dx) >= half_h || fabs(dy) >= half_h) {
      int ib = i / G.bs + (jg / G.bs) * G.nbx;
      unsigned long long local = (unsigned long long)((jg % G.bs) * G.bs + (i % G.bs));
      atomicMin(&sc->err_key, (ERR_CFL << 58) | ((unsigned long long)ib << 24) | local);
    }
    Ht[m] = ht;
    Qx[m] = qx;
    Qy[m] = qy;
  }

  // ---- phase 3: x faces (stepper.cpp:402-447, 496-516) -----------------------
  double px_m[PER], px_a[PER], px_c[PER];  // (W.fm-E.fm), (W.fnr-E.fnl), (W.ft-E.ft)
  double outflow = 0.0;
  auto lc = [&](int s, int dir) {
    LineCell L;
    L.depth = R[F_D * RREG + s];
    L.eta = R[F_E * RREG + s];
    L.un = R[(dir == 0 ? F_U : F_V) * RREG + s];
    L.ut = R[(dir == 0 ? F_V : F_U) * RREG + s];
    L.sh = R[(dir == 0 ? F_SX : F_SY) * RREG + s];
    return L;
  };
  for (int c = tid; c < (BX + 1) * BY; c += NTHR) {
    int fx = c % (BX + 1), y = c / (BX + 1);
    int f = i0 + fx, r = r0 + y;
    FaceRec rec;
    rec.fm = rec.fnl = rec.fnr = rec.ft = 0.0;
    if (f <= G.nx && r < G.r1) {
      int jg = G.jg0 + r;
      int sa = (fx + 1) + (y + 2) * RX;  // cell f-1
      if (f == 0 || f == G.nx) {
        bool lo = f == 0;
        int se = lo ? sa + 1 : sa;
        double H = R[F_D * RREG + se];
        bool wet = H > P.eps;
        rec = boundary_face(wet, H, R[F_U * RREG + se], R[F_V * RREG + se], lo,
                            lo ? G.west_refl : G.east_refl, P.g);
        outflow += lo ? -rec.fm : rec.fm;
      } else {
        bool has_m = f - 2 >= 0, has_p = f + 1 < G.nx;
        rec = interior_face(lc(sa - 1, 0), has_m, lc(sa, 0), R[F_B * RREG + sa], lc(sa + 1, 0),
                            R[F_B * RREG + sa + 1], lc(sa + 2, 0), has_p, P.eps, P.g, P.h);
        if (!face_finite(rec)) atomicMin(&sc->err_key, fused_flux_key(G, A.bflag, 0, jg, f));
      }
    }
    FB[0 * NF + c] = rec.fm;
    FB[1 * NF + c] = rec.fnl;
    FB[2 * NF + c] = rec.fnr;
    FB[3 * NF + c] = rec.ft;
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    int c = tid + m * NTHR;
    int x = c % BX, y = c / BX;
    int w = x + y * (BX + 1), e = w + 1;
    px_m[m] = FB[0 * NF + w] - FB[0 * NF + e];
    px_a[m] = FB[2 * NF + w] - FB[1 * NF + e];
    px_c[m] = FB[3 * NF + w] - FB[3 * NF + e];
  }
  __syncthreads();

  // ---- phase 4: y faces (stepper.cpp:449-494, 518-538) -----------------------
  for (int c = tid; c < BX * (BY + 1); c += NTHR) {
    int x = c % BX, fy = c / BX;
    int i = i0 + x, rf = r0 + fy;  // face between local rows rf-1 and rf
    int jf = G.jg0 + rf;           // global face index
    FaceRec rec;
    rec.fm = rec.fnl = rec.fnr = rec.ft = 0.0;
    bool owned_face = i < G.nx && (rf < G.r1 || (rf == G.r1 && fy <= BY));
    if (owned_face && rf <= G.r1) {
      int sa = (x + 2) + (fy + 1) * RX;  // cell rf-1
      if (jf == 0 || jf == G.ny) {
        bool lo = jf == 0;
        int se = lo ? sa + RX : sa;
        double H = R[F_D * RREG + se];
        bool wet = H > P.eps;
        rec = boundary_face(wet, H, R[F_V * RREG + se], R[F_U * RREG + se], lo,
                            lo ? G.south_refl : G.north_refl, P.g);
        outflow += lo ? -rec.fm : rec.fm;
      } else {
        bool has_m = jf - 2 >= 0, has_p = jf + 1 < G.ny;
        rec = interior_face(lc(sa - RX, 1), has_m, lc(sa, 1), R[F_B * RREG + sa],
                            lc(sa + RX, 1), R[F_B * RREG + sa + RX], lc(sa + 2 * RX, 1), has_p,
                            P.eps, P.g, P.h);
        if (!face_finite(rec)) atomicMin(&sc->err_key, fused_flux_key(G, A.bflag, 1, i, jf));
      }
    }
    FB[0 * NF + c] = rec.fm;
    FB[1 * NF + c] = rec.fnl;
    FB[2 * NF + c] = rec.fnr;
    FB[3 * NF + c] = rec.ft;
  }
  __syncthreads();

  // ---- phase 5: accumulate (stepper.cpp:540-566) + final (628-659) ---------
  double deficit = 0.0;
  const double dt_h = tau / P.h;
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    int c = tid + m * NTHR;
    int x = c % BX, y = c / BX;
    int i = i0 + x, r = r0 + y;
    if (i >= G.nx || r >= G.r1) continue;
    int jg = G.jg0 + r;
    int s = (x + 2) + (y + 2) * RX;
    size_t k = (size_t)i + (size_t)r * nx;
    double Hn = R[F_HN * RREG + s], qxn = R[F_QX * RREG + s], qyn = R[F_QY * RREG + s];
    int lb = i / G.bs + (jg / G.bs - G.bj0) * G.nbx;
    bool flux_on = !G.skip || (A.bflag[lb] & 2);
    if (!flux_on) {  // block skipped by the reference: state unchanged
      A.Ho[k] = Hn;
      A.HUxo[k] = qxn;
      A.HUyo[k] = qyn;
      continue;
    }
    int sf = x + y * BX, nf_ = sf + BX;  // S and N face of the cell
    double py_m = FB[0 * NF + sf] - FB[0 * NF + nf_];
    double py_a = FB[2 * NF + sf] - FB[1 * NF + nf_];  // S.fnr - N.fnl
    double py_c = FB[3 * NF + sf] - FB[3 * NF + nf_];  // S.ft - N.ft
    double d = R[F_D * RREG + s];
    bool wet = d > P.eps;
    double cx = 0.0, cy = 0.0;
    if (wet) {
      auto nb = [&](bool in, int q) {
        Nbr o;
        o.in = in;
        o.depth = R[F_D * RREG + q];
        o.eta = R[F_E * RREG + q];
        o.ux = 0.0;
        o.uy = 0.0;
        return o;
      };
      double eta_c = R[F_E * RREG + s];
      double gx = eta_grad_comp(nb(i > 0, s - 1), nb(i + 1 < G.nx, s + 1), eta_c, P);
      double gy = eta_grad_comp(nb(jg > 0, s - RX), nb(jg + 1 < G.ny, s + RX), eta_c, P);
      double gh = (P.g * d) * P.h;
      cx = gh * gx;
      cy = gh * gy;
    }
    double Fh = px_m[m] + py_m;
    double Fvx = (px_a[m] + py_c) + cx;
    double Fvy = (py_a + px_c[m]) + cy;
    double sgn_ = 0.0;
    if (nsrc > 0) sgn_ = cell_sigma_only(A.src, sig_n, nsrc, i, jg);
    bool act = Hn > P.eps || sgn_ != 0.0;
    double H1, qx, qy, dfc;
    final_cell(act ? Ht[m] : Hn, act ? Qx[m] : qxn, act ? Qy[m] : qyn, Fh, Fvx, Fvy, dt_h, P.eps,
               H1, qx, qy, dfc);
    deficit += dfc;
    A.Ho[k] = H1;
    A.HUxo[k] = qx;
    A.HUyo[k] = qy;
  }
  if (tid == 0) A.tile_same[tile] = 0;

  // ---- per-tile diagnostic partials (deterministic) ------------------------
  __shared__ double s_red[3][NTHR / 32];
  double v3[3] = {deficit, srcvol, outflow};
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    double v = v3[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) s_red[q][tid >> 5] = v;
  }
  __syncthreads();
  if (tid < 3) {
    double v = 0.0;
    for (int w = 0; w < NTHR / 32; ++w) v += s_red[tid][w];
    A.part[3 * tile + tid] = v;
  }
}

// k_finish: diagnostics over tiles in tile order (deterministic), commit t.
__global__ void k_finish(Geo G, const double* part, int ntiles, StepScalars* sc, double area,
                         double h) {
  __shared__ double s[3][256];
  bool stop = stopped(sc);
  double v[3] = {0.0, 0.0, 0.0};
  int per = (ntiles + blockDim.x - 1) / blockDim.x;
  int a = threadIdx.x * per, e = min(a + per, ntiles);
  if (!stop)
    for (int t = a; t < e; ++t) {
      v[0] += part[3 * t + 0];
      v[1] += part[3 * t + 1];
      v[2] += part[3 * t + 2];
    }
  for (int q = 0; q < 3; ++q) s[q][threadIdx.x] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
    if (stop) {
      if (sc->fail_step < 0) sc->fail_step = sc->steps_done;
      return;
    }
    double w[3] = {0.0, 0.0, 0.0};
    for (int t = 0; t < (int)blockDim.x; ++t)
      for (int q = 0; q < 3; ++q) w[q] += s[q][t];
    sc->deficit = w[0] * area;
    sc->srcvol = w[1] * area;
    sc->outflow = (w[2] * sc->tau) * h;
    sc->t += sc->tau;  // stepper.cpp:703
    sc->steps_done += 1;
  }
}

StepArgs step_args(swf_ctx* c) {
  StepArgs A;
  int cur = c->cur, nxt = 1 - c->cur;
  A.H = c->H[cur];
  A.HUx = c->HUx[cur];
  A.HUy = c->HUy[cur];
  A.b = c->b;
  A.nf = c->nf;
  A.fpx = c->fpx;
  A.fpy = c->fpy;
  A.Ho = c->H[nxt];
  A.HUxo = c->HUx[nxt];
  A.HUyo = c->HUy[nxt];
  A.src = c->d_src;
  A.sig = c->d_sig;
  A.bflag = c->d_bflag;
  A.tile_act = c->d_tile_act;
  A.tile_same = c->d_tile_same;
  A.part = c->d_part;
  A.sc = c->d_sc;
  return A;
}

constexpr size_t step_smem() {
  return (size_t)(F_NUM * RREG + 4 * ((BX + 1) * BY > BX * (BY + 1) ? (BX + 1) * BY
                                                                     : BX * (BY + 1))) *
         sizeof(double);
}

void ev(swf_ctx* c, int i) {
  if (!c->timing) return;
  if (c->tslots > 0)
    cudaEventRecord(c->tev[(size_t)(c->tstep % c->tslots) * 6 + i], c->stream);
  else
    cudaEventRecord(c->ev[i], c->stream);
}

// rows k_forces must cover: owned rows plus 2 ghost rows on each interior side
void forces_rows(const swf_ctx* c, int& ra0, int& ra1) {
  ra0 = c->geo.r0 - (c->geo.r0 >= 2 ? 2 : c->geo.r0);
  ra1 = c->geo.r1 + (c->geo.rows - c->geo.r1 >= 2 ? 2 : c->geo.rows - c->geo.r1);
  // a ghost row at the local edge has no outer neighbour row: keep one
  // layer of the ghost band as pure input
  if (ra0 < c->geo.r0 && ra0 == 0) ra0 = 1;
  if (ra1 > c->geo.r1 && ra1 == c->geo.rows) ra1 = c->geo.rows - 1;
}

}  // namespace

int launch_begin(swf_ctx* c, double dt_cap) {
  k_begin<<<1, 1, 0, c->stream>>>(c->geo, c->d_src, c->d_ht, c->d_hq, c->d_wt, c->d_wv, c->d_sig,
                                  c->d_sc, dt_cap);
  return cuda_check(c, cudaGetLastError(), "k_begin");
}

int launch_mask(swf_ctx* c) {
  const Geo& G = c->geo;
  int nbl = G.nbx * (G.bj1 - G.bj0);
  if (nbl > 0)
    k_mask<<<(nbl + 127) / 128, 128, 0, c->stream>>>(G, c->H[c->cur], c->d_src, c->d_sig,
                                                      c->d_interior, c->d_halo, c->d_bflag,
                                                      c->d_sc);
  int nt = G.tiles_x * G.tiles_y;
  if (nt > 0) k_tiles<<<(nt + 127) / 128, 128, 0, c->stream>>>(G, c->d_bflag, c->d_tile_act);
  return cuda_check(c, cudaGetLastError(), "k_mask");
}

int launch_tau(swf_ctx* c, double dt_cap) {
  k_tau<<<1, 1, 0, c->stream>>>(c->geo, c->d_src, c->d_ht, c->d_hq, c->d_wt, c->d_wv, c->d_sig,
                                c->d_sc, dt_cap, -1.0);
  return cuda_check(c, cudaGetLastError(), "k_tau");
}

int launch_mid(swf_ctx* c, double tau) {
  k_mid<<<1, 1, 0, c->stream>>>(c->geo, c->d_src, c->d_ht, c->d_hq, c->d_wt, c->d_wv, c->d_sig,
                                c->d_sc, tau);
  return cuda_check(c, cudaGetLastError(), "k_mid");
}

int fused_enqueue_phase1(swf_ctx* c, double dt_cap) {
  const Geo& G = c->geo;
  int rc;
  ev(c, 0);
  if ((rc = launch_begin(c, dt_cap))) return rc;
  if ((rc = launch_mask(c))) return rc;
  ev(c, 1);
  int ra0, ra1;
  forces_rows(c, ra0, ra1);
  int txa = (G.nx + AX - 1) / AX, tya = (ra1 - ra0 + AY - 1) / AY;
  if (txa * tya > 0)
    k_forces<<<txa * tya, NTHR, 0, c->stream>>>(G, ra0, ra1, txa, c->H[c->cur], c->HUx[c->cur],
                                                c->HUy[c->cur], c->b, c->nf, c->d_src, c->d_sig,
                                                c->fpx, c->fpy, c->d_sc);
  ev(c, 2);
  return cuda_check(c, cudaGetLastError(), "k_forces");
}

int fused_enqueue_phase2(swf_ctx* c, double dt_cap, double global_speed) {
  const Geo& G = c->geo;
  k_tau<<<1, 1, 0, c->stream>>>(G, c->d_src, c->d_ht, c->d_hq, c->d_wt, c->d_wv, c->d_sig,
                                c->d_sc, dt_cap, global_speed);
  ev(c, 3);
  int nt = G.tiles_x * G.tiles_y;
  if (nt > 0) k_step<<<nt, NTHR, step_smem(), c->stream>>>(G, step_args(c));
  ev(c, 4);
  k_finish<<<1, 256, 0, c->stream>>>(G, c->d_part, nt, c->d_sc, c->h * c->h, c->h);
  ev(c, 5);
  if (c->timing && c->tslots > 0) ++c->tstep;
  c->cur = 1 - c->cur;  // optimistic; rolled back by the caller on failure
  return cuda_check(c, cudaGetLastError(), "k_step");
}

int fused_enqueue_phase2(swf_ctx* c, double dt_cap) { return fused_enqueue_phase2(c, dt_cap, -1.0); }

int fused_enqueue_step(swf_ctx* c, double dt_cap) {
  int rc = fused_enqueue_phase1(c, dt_cap);
  if (rc) return rc;
  return fused_enqueue_phase2(c, dt_cap, -1.0);
}

size_t fused_tile_bytes() { return step_smem(); }

// Kernel attributes must be set outside stream capture (a CUDA graph does not
// record cudaFuncSetAttribute), so contexts call this at creation.
int fused_prepare(swf_ctx* c) {
  cudaError_t e = cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)step_smem());
  return cuda_check(c, e, "k_step shared-memory attribute");
}

}  // namespace swf
