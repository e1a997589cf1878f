// swf_fused.cu — the FUSED fast path of one CSPH-TVD step on sm_100a.
//
// One step on the context's stream (captured in a CUDA graph for swf_run):
//   k_begin        1 thread   sources sigma_s(t_n), wind(t_n), counters
//   k_flist        1 thr/tile dry-neighbourhood rule -> k_forces work list
//   k_forces_list  persistent K1 + K2 + K3 per listed 32x16 tile: the block
//                             mask of its B-blocks (block.cpp:16-61) and the
//                             tile flags, forces on wet cells (f - f_fric
//                             only), the CFL speed (shuffles + one atomicMax)
//   k_forces_redo  148 CTAs   tiles with a rejected speculative division, exact
//   k_tau          1 thread   tau = min(dt_max, K h / speed, dt_cap); t_mid,
//                             wind(t_mid), sigma_s(t_mid) (stepper.cpp:256-266, 311-319)
//   k_slist        1 thr/tile k_step work list (active or not-yet-copied tiles)
//   k_step_list    persistent K4..K8 fused per tile: predictor on the tile + 2-cell
//                             halo, mid forces + corrector on owned cells, minmod
//                             slopes once per cell and direction, x- then y-face
//                             HLL fluxes in shared memory, accumulate, final
//                             update into the other state buffer (ping-pong)
//   k_step_redo    148 CTAs   tiles with a rejected speculative division, exact
//   k_reduce       148 CTAs   fixed-order diagnostics partials; k_finish commits t
// (block sizes that do not divide 16 use a separate k_mask/k_tiles pair and
// one CTA per tile; strip contexts split k_forces around the halo exchange).
//
// HBM traffic per wet cell-update: k_forces reads H,HUx,HUy,b (+n) and writes
// 2 doubles; k_step reads H,HUx,HUy,b,f' (+n) and writes H,HUx,HUy — ≈120 B
// against the 56 B compulsory minimum; the FP64 pipe and its dependency
// chains, not HBM, bound this path.  Dry tiles cost one
// thread in each list kernel and, once after they go dry, one copy between
// the ping-pong buffers.
#include <cuda_runtime.h>

#include <vector>

#include "swf_internal.cuh"

namespace swf {
namespace {

// ---- tiles -----------------------------------------------------------------
constexpr int BX = 32, BY = 16;  // tile of owned cells (k_forces and k_step)
constexpr int AX = BX, AY = BY;
constexpr int AREGX = AX + 2, AREGY = AY + 2, AREG = AREGX * AREGY;  // 1-cell halo
constexpr int RX = BX + 4, RY = BY + 4, RREG = RX * RY;              // 2-cell halo
constexpr int NTHR = 256;  // k_reduce, k_scatter_host, k_ingest_hu, k_finish
#ifndef SWF_FORCES_THREADS
#define SWF_FORCES_THREADS 128
#endif
constexpr int FTHR = SWF_FORCES_THREADS;  // k_forces (whole warps)
constexpr int MAXBF = 64;  // B-block flags of one tile staged in shared memory
constexpr int HALO_ROWS = SWF_HALO;  // ghost rows per interior strip side (swf.h)
#ifndef SWF_STEP_THREADS
#define SWF_STEP_THREADS 256
#endif
constexpr int STHR = SWF_STEP_THREADS;  // k_step (a multiple of 32)
static_assert(STHR % 32 == 0, "k_step threads must be whole warps");
constexpr int RED_CTAS = 148;
constexpr int NPART_ALLOC = 5;  // doubles per tile in d_part (see k_reduce)
#ifndef SWF_PHASE_UNROLL  // unroll factor of k_step's region / slope / face loops (1: rolled)
#define SWF_PHASE_UNROLL 1
#endif
#define SWF_PRAGMA_(x) _Pragma(#x)
#define SWF_UNROLL_(n) SWF_PRAGMA_(unroll n)
#define SWF_PHASE_LOOP SWF_UNROLL_(SWF_PHASE_UNROLL)
#ifndef SWF_TMA_L2PROMO  // L2 promotion of the region tensor copies (0 none, 1 64B, 2 128B, 3 256B)
#define SWF_TMA_L2PROMO 3
#endif
#ifndef SWF_TMA  // slim k_step: the region's H, HUx, HUy, b tiles by TMA (cp.async.bulk.tensor)
#define SWF_TMA 1
#endif
#ifndef SWF_EPI_ONEBAR  // k_step epilogue: the partials' barrier is the acceptance barrier
#define SWF_EPI_ONEBAR 1
#endif
#ifndef SWF_OWN_FB  // slim k_step: the owned cells' step-start state kept in the face planes for phase 2
#define SWF_OWN_FB 1
#endif
#ifndef SWF_P2_ROLLED  // k_step phase 2 as a rolled loop, the Lagrangian state parked in the output buffers
#define SWF_P2_ROLLED 1
#endif
#ifndef SWF_GRAD_SHARE  // k_step's mid forces hand the half-step eta gradient to its final update
#define SWF_GRAD_SHARE 1
#endif
#ifndef SWF_LAMBDA_SHARE  // k_forces hands lambda(H_n, n) of the wet cells to k_step
#define SWF_LAMBDA_SHARE 1
#endif
#ifndef SWF_XDIAG_SRC  // developer A/B switches of the exact-volume term stores
#define SWF_XDIAG_SRC 1
#endif
#ifndef SWF_XDIAG_DEF
#define SWF_XDIAG_DEF 1
#endif
#ifndef SWF_STEP_SLIM  // k_step's slim region (see the plane enum); -DSWF_STEP_SLIM=0: the full one
#define SWF_STEP_SLIM 1
#endif
#ifndef SWF_SPLIT  // the split step (k_lag + k_flux), measured and opt-in; needs SWF_STEP_SLIM=0
#define SWF_SPLIT 0
#endif
#ifndef SWF_STEP_MINB
#define SWF_STEP_MINB (SWF_STEP_SLIM ? 4 : 3)  // CTAs per SM the register budget of k_step targets
#endif
#ifndef SWF_FORCES_MINB
// 9 CTAs of 128 threads per SM caps k_forces at 56 registers; ptxas then
// spills 12-20 B per thread in k_forces_list / k_forces_redo (L1-resident).
// Measured as the best trade-off (profiles/README.md, rounds 2t-2v: 128 x 9
// 3.125 ms, 128 x 8 3.134, 128 x 7 3.27, 256 x 6 3.58).
#define SWF_FORCES_MINB 9
#endif


// Developer instrumentation (-DSWF_PHASE_TIMING): per-phase cycles of
// k_step summed over CTAs (thread 0 of each CTA; phases end at barriers).
#ifdef SWF_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[16];
#define PHASE_MARK(i)                                                         \
  do {                                                                        \
    if (threadIdx.x == 0) {                                                   \
      long long t2_ = clock64();                                              \
      atomicAdd(&g_phase_cycles[i], (unsigned long long)(t2_ - t_ph));        \
      t_ph = t2_;                                                             \
    }                                                                         \
  } while (0)
#else
#define PHASE_MARK(i) \
  do {                \
  } while (0)
#endif

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
  sc->redo_n[0] = 0;
  sc->redo_n[1] = 0;
  sc->redo_n[2] = 0;
  sc->list_n[0] = sc->list_n[1] = 0;
  sc->list_take[0] = sc->list_take[1] = sc->list_take[2] = 0;
  for (int q = 0; q < SPEED_SLOTS; ++q) sc->speed_slots[q] = 0ull;
  sc->lag_act = 0;
  sc->flux_act = 0;
  sc->dt_cap = dt_cap;
  sc->host_writes = 0ull;
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
// gspeed (device pointer, may be null) overrides both: the allreduced speed
// of an asynchronous multi-strip step, read without a host round trip.
__global__ void k_tau(Geo G, const DevSrc* src, const double* ht, const double* hq,
                      const double* wt, const double* wv, double* sig, StepScalars* sc,
                      double dt_cap, double global_speed, const double* gspeed) {
  sc->mask_fresh = 0;  // k_flist has consumed it
  sc->step_open = 0;
  if (stopped(sc)) return;
  unsigned long long mb = sc->speed_bits;
  for (int q = 0; q < SPEED_SLOTS; ++q) mb = sc->speed_slots[q] > mb ? sc->speed_slots[q] : mb;
  sc->speed_bits = mb;
  if (gspeed && dbits(*gspeed) == SPEED_STOP_BITS) {  // another strip has stopped
    atomicMin(&sc->err_key, ERR_PEER << 58);
    return;
  }
  double speed = gspeed ? *gspeed : (global_speed >= 0.0 ? global_speed : bitsd(mb));
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
  if (dt_cap < 0.0) dt_cap = sc->dt_cap_dev;  // set on the device (nested subcycling)
  if (dt_cap > 0.0) tau = smin(tau, dt_cap);
  sc->tau = tau;
  mid_scalars(G, src, ht, hq, wt, wv, sig, sc, tau);
  sc->step_open = 1;
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
  if (stopped(sc)) return;  // (see k_flist)
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
__global__ void k_tiles(Geo G, const unsigned char* bflag, unsigned char* tile_act,
                        const StepScalars* sc) {
  if (stopped(sc)) return;  // (see k_flist)
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


// Bitmask of the source specs whose rectangle meets the global cell box
// [ci0, ci1] x [cj0, cj1] (at most 32 specs; more -> all bits).  Cells outside
// a spec's rectangle get nothing from it, so evaluating only the masked
// specs, in spec order, reproduces the full per-cell sums exactly.
__device__ __forceinline__ unsigned src_mask_for(const Geo& G, const DevSrc* src, int ci0, int ci1,
                                                 int cj0, int cj1) {
  if (G.nsrc > 32) return 0xffffffffu;
  unsigned m = 0;
  for (int s = 0; s < G.nsrc; ++s) {
    const DevSrc& d = src[s];
    if (d.i0 <= ci1 && d.i1 >= ci0 && d.j0 <= cj1 && d.j1 >= cj0) m |= 1u << s;
  }
  return m;
}

#ifndef SWF_SRC_ROLLED  // keep the source lookup loops rolled (rare path, compact code)
#define SWF_SRC_ROLLED 1
#endif
__device__ __forceinline__ double msrc(const Geo& G, const DevSrc* src, const double* sig,
                                       unsigned mask, int i, int jg, double& vx, double& vy) {
  double s = 0.0;
  if (!mask) return s;
#if SWF_SRC_ROLLED
#pragma unroll 1
#endif
  for (int m = 0; m < G.nsrc; ++m) {
    if (G.nsrc <= 32 && !((mask >> m) & 1u)) continue;
    const DevSrc& d = src[m];
    if (i >= d.i0 && i <= d.i1 && jg >= d.j0 && jg <= d.j1) {
      s += sig[m];
      vx = d.vx;
      vy = d.vy;
    }
  }
  return s;
}

__device__ __forceinline__ double msig(const Geo& G, const DevSrc* src, const double* sig,
                                       unsigned mask, int i, int jg) {
  double vx, vy;
  return msrc(G, src, sig, mask, i, jg, vx, vy);
}

// Neighbour view over shared-memory planes (depth, eta, ux, uy at index q),
// read where the force helpers use them: holding the four neighbours' values
// in registers across cell_forces spilled them (k_forces at its 40-register
// budget, k_step's phase 2).
struct SNbr {
  bool in;
  const double *d, *e, *u, *v;
  int q;
  __device__ __forceinline__ double dep() const { return d[q]; }
  __device__ __forceinline__ double et() const { return e[q]; }
  __device__ __forceinline__ double vx() const { return u[q]; }
  __device__ __forceinline__ double vy() const { return v[q]; }
};

// ---------------------------------------------------------------------------
// Speculative division.  The tile bodies are templates on SPEC.  With SPEC,
// every rdiv returns its fast-path quotient and clears the thread's flag
// `sok` when that quotient was not accepted (tiny or denormal operands), so
// the bodies carry no slow-path branches; a tile with any rejected division
// is appended to a redo list instead of publishing its CFL speed or error,
// and a second, exact (SPEC = false) launch recomputes the listed tiles from
// the same inputs.  Every result is therefore the exact one, bit for bit.
// ---------------------------------------------------------------------------
#ifndef SWF_SPECULATE
#define SWF_SPECULATE 1
#endif
#ifndef SWF_TILE_LISTS
#define SWF_TILE_LISTS 1  // work lists + persistent CTAs instead of one CTA per tile
#endif
#define SP (SPEC ? &sok : (bool*)nullptr)

// ---------------------------------------------------------------------------
// k_forces: K1 + K2 + K3 on a BX x BY tile with a 1-cell halo.
//  * K1 (fused when the block size divides 16): interior / clamped-ring wet
//    counts of the tile's B-blocks (block.cpp:16-61), block flags, tile flags.
//  * K2: forces on wet cells; stores f' = (fx - fric_x, fy - fric_y), the only
//    K2 output the predictor needs (stepper.cpp:283-284).
//  * K3: the CFL speed of wet cells (stepper.cpp:233-254), shuffle max and
//    one atomicMax per CTA.
// Tile rows tr in [tr_lo, tr_hi) relative to the owned rows; forces cover
// local rows [ra0, ra1) (owned + 2 ghost rows per interior strip side).
// ---------------------------------------------------------------------------
struct ForcesArgs {
  const double* __restrict__ H;
  const double* __restrict__ HUx;
  const double* __restrict__ HUy;
  const double* __restrict__ b;
  const double* __restrict__ nf;
  const DevSrc* src;
  const double* sig;
  double* __restrict__ fpx;
  double* __restrict__ fpy;
  double* __restrict__ lamn;  // SWF_LAMBDA_SHARE: lambda(H_n, n) of each wet cell
  int* interior;
  int* halo;
  unsigned char* bflag;
  unsigned char* tile_act;
  StepScalars* sc;
  double* cnt_part;  // per-tile diagnostics partials: slots 3, 4 = block counts
  const unsigned char* tile_prev;  // tile flags of the previous step
  const unsigned* tile_srcm;       // per owned tile (see StepArgs)
  int* redo;                       // tiles whose speculative divisions were rejected
  int* list;                       // work list of k_flist / k_forces_list
  int ra0, ra1, tr_lo, do_mask;
  int lr0, lr1;                    // tile rows the work list covers (strips: ghost rows too)
};

// redo-list entries: tile column + (tile row + REDO_ROW0) * tiles_x
constexpr int REDO_ROW0 = 4;

// presel: the tile comes from the work list k_flist built, which already
// applied the dry-neighbourhood rule below.
template <bool SPEC>
__device__ __forceinline__ void forces_tile(const Geo& G, const ForcesArgs& A, const int tx,
                                            const int tr, const bool presel = false) {
  __shared__ double s_d[AREG], s_e[AREG], s_u[AREG], s_v[AREG];
  __shared__ unsigned char s_w[AREG];
  __shared__ int s_cnt[3];
  __shared__ unsigned s_srcm;
  __shared__ unsigned long long s_max[FTHR / 32];
  StepScalars* sc = A.sc;
  if (__syncthreads_or(stopped(sc))) return;
  bool sok = true;  // every speculative division of this thread accepted
  const PhysConst& P = G.P;  // reciprocals refined at context creation (fused_prepare)
  const int tid = threadIdx.x;
  const int i0 = tx * BX, rr0 = G.r0 + tr * BY;
  const size_t nx = G.nx;
  // mask rows (owned rows only)
  const bool mask_tile = A.do_mask && tr >= 0 && tr < G.tiles_y;
  const bool own_row = tr >= 0 && tr < G.tiles_y;
  if (tid == 0)
    s_srcm = own_row ? A.tile_srcm[tx + tr * G.tiles_x]
                     : src_mask_for(G, A.src, i0 - 1, i0 + BX, G.jg0 + rr0 - 1, G.jg0 + rr0 + BY);
  // Dry neighbourhood: if this tile and its 8 neighbours had no flux-active
  // block in the previous step, k_step left all their cells untouched, so
  // this tile's block counts, flags and (empty) forces are unchanged: skip.
  // Not across a strip boundary (ghost rows change by exchange) and not near
  // a source (sigma(t) can switch a marker on).  Threads 0..8 read one
  // neighbour flag each.
  const bool may_skip = !presel && mask_tile && G.skip && sc->mask_valid &&
                        (tr > 0 || G.r0 == 0) && (tr < G.tiles_y - 1 || G.r1 == G.rows);
  bool busy = !may_skip;
  if (may_skip && tid < 9) {
    int x2 = tx + tid % 3 - 1, y2 = tr + tid / 3 - 1;
    if (x2 >= 0 && x2 < G.tiles_x && y2 >= 0 && y2 < G.tiles_y)
      busy = A.tile_prev[x2 + y2 * G.tiles_x] != 0;
  }
  busy = __syncthreads_or(busy);
  const unsigned srcm = s_srcm;
  if (!busy && !srcm) {
    if (tid == 0) A.tile_act[tx + tr * G.tiles_x] = 0;
    return;
  }
  // forces rows of this tile
  const int fa = max(rr0, A.ra0), fb = min(rr0 + BY, A.ra1);

  // ---- region state (all loads issued together) + wet flags (K1) ------------
  bool anywet = false;
  for (int c = tid; c < AREG; c += FTHR) {
    int i = i0 - 1 + c % AREGX, r = rr0 - 1 + c / AREGX;
    double d = 0.0, mx = 0.0, my = 0.0, bb = 0.0;
    unsigned char w = 0;
    if (i >= 0 && i < G.nx && r >= 0 && r < G.rows) {
      size_t k = (size_t)i + (size_t)r * nx;
      d = A.H[k];
      mx = A.HUx[k];
      my = A.HUy[k];
      bb = A.b[k];
      bool wet = d > P.eps;
      w = wet || (srcm && msig(G, A.src, A.sig, srcm, i, G.jg0 + r) != 0.0);
      int x = c % AREGX - 1, y = c / AREGX - 1;
      if (wet && x >= 0 && x < BX && y >= 0 && y < BY && r >= fa && r < fb) anywet = true;
    }
    s_d[c] = d;
    s_u[c] = mx;
    s_v[c] = my;
    s_e[c] = bb;
    s_w[c] = w;
  }
  if (tid < 3) s_cnt[tid] = 0;
  anywet = __syncthreads_or(anywet);

  // ---- K1: block counts of the tile's B-blocks ------------------------------
  // One warp per block: interior cells and the clamped one-cell ring
  // (corners included, block.cpp:36-56) counted with ballots; no atomics on
  // global counters — the per-tile counts go to the diagnostics partials.
  // K1 runs on the first min(nbt, FTHR/32) warps while the others convert
  // the region to eta/velocity (independent: K1 reads only the wet flags;
  // with FTHR = 128 and 16-cell blocks all 4 warps count, then convert)
  // (the mask is fused only when bs divides 16: a power of two, so shifts)
  const int lgb = __ffs(G.bs) - 1;
  const int nbt = mask_tile ? (BX >> lgb) * (BY >> lgb) : 0;
  const int k1w = mask_tile ? min(nbt, FTHR / 32) : 0;
  if (mask_tile) {
    const int bs = G.bs, lgx = 5 - lgb, nbxt = BX >> lgb;  // BX = 32 = 2^5
    const int rend = min(rr0 + BY, G.r1);
    const int lane = tid & 31, warp = tid >> 5;
    for (int blk = warp; blk < nbt; blk += FTHR / 32) {
      int bx = blk & (nbxt - 1), by = blk >> lgx;
      int bi0 = i0 + bx * bs, br0 = rr0 + by * bs;  // block origin (global col, local row)
      if (bi0 >= G.nx || br0 >= rend) continue;
      int bi1 = min(bi0 + bs - 1, G.nx - 1), br1 = min(br0 + bs - 1, rend - 1);
      int wdt = bi1 - bi0 + 1, hgt = br1 - br0 + 1;
      int in = 0, ring = 0;
      const int lg = lgb;
      for (int p = lane; p < bs * bs; p += 32) {
        int px = p & (bs - 1), py = p >> lg;
        if (px < wdt && py < hgt)
          in += s_w[(bi0 + px - (i0 - 1)) + (br0 + py - (rr0 - 1)) * AREGX];
      }
      const int top = wdt + 2, per = 2 * top + 2 * hgt;
      for (int q = lane; q < per; q += 32) {
        int ci, cj;  // global, then clamped into the domain
        if (q < top) {
          ci = bi0 - 1 + q;
          cj = G.jg0 + br0 - 1;
        } else if (q < 2 * top) {
          ci = bi0 - 1 + (q - top);
          cj = G.jg0 + br1 + 1;
        } else {
          int qq = q - 2 * top;
          cj = G.jg0 + br0 + (qq >> 1);
          ci = (qq & 1) ? bi1 + 1 : bi0 - 1;
        }
        ci = min(max(ci, 0), G.nx - 1);
        cj = min(max(cj, 0), G.ny - 1);
        ring += s_w[(ci - (i0 - 1)) + ((cj - G.jg0) - (rr0 - 1)) * AREGX];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        in += __shfl_xor_sync(0xffffffffu, in, o);
        ring += __shfl_xor_sync(0xffffffffu, ring, o);
      }
      if (lane == 0) {
        int lb = (bi0 >> lgb) + (((G.jg0 + br0) >> lgb) - G.bj0) * G.nbx;
        A.interior[lb] = in;
        A.halo[lb] = ring;
        bool l = in > 0, f = l || ring > 0;
        A.bflag[lb] = (l ? 1 : 0) | (f ? 2 : 0);
        if (l) atomicAdd(&s_cnt[0], 1);
        if (f) atomicAdd(&s_cnt[1], 1);
      }
    }
  }

  // ---- region momentum -> eta, velocity ---------------------------------------
  const int vt0 = k1w < FTHR / 32 ? 32 * k1w : 0;  // first thread of the velocity pass
  if (anywet && tid >= vt0) {
    for (int c = tid - vt0; c < AREG; c += FTHR - vt0) {  // pointwise, in place (same c)
      double d = s_d[c];
      double e = d + s_e[c], u = 0.0, v = 0.0;
      if (d > P.eps) {
        Recip Rd = recip_of(d);
        u = rdiv(s_u[c], Rd, SP);
        v = rdiv(s_v[c], Rd, SP);
      }
      s_e[c] = e;
      s_u[c] = u;
      s_v[c] = v;
    }
  }
  __syncthreads();
  if (mask_tile && tid == 0) {
    int t = tx + tr * G.tiles_x;
    A.tile_act[t] = G.skip ? ((s_cnt[0] ? 1 : 0) | (s_cnt[1] ? 2 : 0)) : 3;
    A.cnt_part[5 * (size_t)t + 3] = s_cnt[0];
    A.cnt_part[5 * (size_t)t + 4] = s_cnt[1];
  }
  if (!anywet) return;

  // ---- K2 forces + K3 speed on wet cells ------------------------------------
  double m = 0.0;
  const double wx = sc->wind_n[0], wy = sc->wind_n[1];
  for (int c = tid; c < AX * AY; c += FTHR) {
    int x = c % AX, y = c / AX;
    int i = i0 + x, r = rr0 + y;
    if (i >= G.nx || r < fa || r >= fb) continue;
    int s = (x + 1) + (y + 1) * AREGX;
    double d = s_d[s];
    if (!(d > P.eps)) continue;
    int jg = G.jg0 + r;
    auto nb = [&](bool in, int q) { return SNbr{in, s_d, s_e, s_u, s_v, q}; };
    SNbr W = nb(i > 0, s - 1), E = nb(i + 1 < G.nx, s + 1);
    SNbr S = nb(jg > 0, s - AREGX), N = nb(jg + 1 < G.ny, s + AREGX);
    double sg = 0.0, svx = 0.0, svy = 0.0;
    if (srcm) sg = msrc(G, A.src, A.sig, srcm, i, jg, svx, svy);
    size_t k = (size_t)i + (size_t)r * nx;
    double n = G.has_nfield ? A.nf[k] : G.n_manning;
    double ux = s_u[s], uy = s_v[s];
#if SWF_LAMBDA_SHARE
    const double lam = manning_lambda(d, P.g, n, SP);
    A.lamn[k] = lam;  // the predictor's lambda(H12) when H12 == H_n (no source)
    ForceOut o = cell_forces_lam(d, ux, uy, s_e[s], W, E, S, N, lam, P, G.nwind > 0, wx, wy, sg,
                                 svx, svy, SP, SP);
#else
    ForceOut o = cell_forces(d, ux, uy, s_e[s], W, E, S, N, n, P, G.nwind > 0, wx, wy, sg, svx,
                             svy, SP);
#endif
    A.fpx[k] = o.fx - o.frx;
    A.fpy[k] = o.fy - o.fry;
    m = cfl_speed(m, d, ux, uy, o.fx, o.fy, P.g, P.h, SP);
  }
  unsigned long long bits = dbits(m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long ob = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = ob > bits ? ob : bits;
  }
  if ((tid & 31) == 0) s_max[tid >> 5] = bits;
  const bool any_bad = __syncthreads_or(!sok);  // (also orders the s_max writes)
  const bool redo = SPEC && any_bad;
  if (tid == 0) {
    if (redo) {  // recomputed exactly by k_forces_redo; publish nothing
      A.redo[atomicAdd(&sc->redo_n[0], 1)] = tx + (tr + REDO_ROW0) * G.tiles_x;
    } else {
      unsigned long long mb = 0;
      for (int w = 0; w < FTHR / 32; ++w) mb = s_max[w] > mb ? s_max[w] : mb;
      // spread over SPEED_SLOTS addresses to avoid one contended L2 atomic
      if (mb) atomicMax(&sc->speed_slots[(tx + tr * 7) & (SPEED_SLOTS - 1)], mb);
    }
  }
}

__global__ void __launch_bounds__(FTHR, SWF_FORCES_MINB) k_forces(Geo G, ForcesArgs A) {
  const int tx = blockIdx.x % G.tiles_x, tr = (int)(blockIdx.x / G.tiles_x) + A.tr_lo;
  forces_tile<SWF_SPECULATE != 0>(G, A, tx, tr);
}

// ---- tile work lists (single-context steps) ---------------------------------
// Warp-aggregated append: one atomic per warp and the lanes' entries in lane
// order, so the list keeps the tiles' raster order within each warp (spatial
// neighbours stay close in time and share their halo rows in L2).
__device__ __forceinline__ void append_ordered(int* list, int* n, bool take, int t) {
  const unsigned m = __ballot_sync(0xffffffffu, take);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(n, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (take) list[base + __popc(m & ((1u << lane) - 1u))] = t;
}

// k_flist: one thread per tile applies the dry-neighbourhood rule of
// forces_tile and appends the tiles k_forces must visit to A.list; the
// skipped ones get their flag cleared exactly as forces_tile would.  A
// persistent k_forces_list grid then takes list entries off an atomic
// counter, so the ~60 % of C3 tiles that are dry cost one thread, not a CTA.
__global__ void k_flist(Geo G, ForcesArgs A) {
  const int nt = G.tiles_x * (A.lr1 - A.lr0);
  const int t = blockIdx.x * blockDim.x + threadIdx.x;  // list index: relative to row lr0
  StepScalars* sc = A.sc;
  // a stopped context's remaining steps of a batch must not touch the tile
  // flags or grow the list (k_begin, which resets it, did not run)
  if (stopped(sc)) return;
  const int tx = t % G.tiles_x, tr = t / G.tiles_x + A.lr0;
  // a strip's ghost tile rows and the tile rows next to its edges are always
  // visited (their halo changes by exchange), like forces_tile's own rule
  const bool own = tr >= 0 && tr < G.tiles_y;
  const bool edge = !own || (tr == 0 && G.r0 > 0) || (tr == G.tiles_y - 1 && G.r1 < G.rows);
  const int tt = own ? tx + tr * G.tiles_x : 0;  // owned-tile index
  const bool valid = t < nt;  // every lane reaches the warp-wide append
  // host-buffer step: k_mask/k_tiles already flagged this state, so a tile
  // whose blocks have no wet cell in their interiors or rings (its forces
  // region is dry) is skipped outright, its block counts zero
  const bool fresh = A.do_mask && G.skip && sc->mask_fresh;
  bool busy;
  if (edge) {
    busy = valid;
  } else if (fresh) {
    busy = valid && (A.tile_act[tt] != 0 || A.tile_srcm[tt] != 0);
  } else {
    busy = valid && (!(A.do_mask && G.skip && sc->mask_valid) || A.tile_srcm[tt] != 0);
    for (int q = 0; q < 9 && valid && !busy; ++q) {
      int x2 = tx + q % 3 - 1, y2 = tr + q / 3 - 1;
      if (x2 >= 0 && x2 < G.tiles_x && y2 >= 0 && y2 < G.tiles_y)
        busy = A.tile_prev[x2 + y2 * G.tiles_x] != 0;
    }
  }
  if (valid && !busy) {  // (never an edge or ghost tile)
    A.tile_act[tt] = 0;
    if (fresh) {
      A.cnt_part[5 * (size_t)tt + 3] = 0.0;
      A.cnt_part[5 * (size_t)tt + 4] = 0.0;
    }
  }
  append_ordered(A.list, &sc->list_n[0], busy, t);
}

__global__ void __launch_bounds__(FTHR, SWF_FORCES_MINB) k_forces_list(Geo G, ForcesArgs A) {
  __shared__ int s_next;
  StepScalars* sc = A.sc;
  const int n = *(volatile int*)&sc->list_n[0];
  while (true) {
    if (threadIdx.x == 0) s_next = atomicAdd(&sc->list_take[0], 1);
    __syncthreads();
    const int q = s_next;
    __syncthreads();
    if (q >= n) break;
    const int t = A.list[q];
    forces_tile<SWF_SPECULATE != 0>(G, A, t % G.tiles_x, t / G.tiles_x + A.lr0, true);
    __syncthreads();
  }
}

// the tiles with a rejected speculative division, recomputed exactly
__global__ void __launch_bounds__(FTHR, SWF_FORCES_MINB) k_forces_redo(Geo G, ForcesArgs A) {
  const int n = *(volatile int*)&A.sc->redo_n[0];
  for (int q = blockIdx.x; q < n; q += gridDim.x) {
    int e = A.redo[q];
    forces_tile<false>(G, A, e % G.tiles_x, e / G.tiles_x - REDO_ROW0);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// k_step: K4..K8 fused over a BX x BY tile.
// ---------------------------------------------------------------------------

// shared-memory fields of the 2-cell-halo region (RX x RY), half-step view
#if SWF_STEP_SLIM
// slim region (the default): depth, velocities and bed only -- eta = d + b
// and the shifts 0.5*tau*u recomputed at the point of use with the stored
// planes' own expressions (bit-identical), the step-start state, f', n and
// lambda read from global memory -- for 4 CTAs of 256 threads per SM (54 KB
// of shared memory, 64 registers): k_step 11.0 -> 10.5 ms on C3 (the full
// region, 76 KB and 80 registers, fits 3; profiles/README.md round 3)
enum { F_D = 0, F_U, F_V, F_B, F_NUM };
#else
enum { F_D = 0, F_E, F_U, F_V, F_SX, F_SY, F_B, F_NUM };
#endif
constexpr int NSL = (BX + 2) * BY > BX * (BY + 2) ? (BX + 2) * BY : BX * (BY + 2);  // slopes
constexpr int NFC = (BX + 1) * BY > BX * (BY + 1) ? (BX + 1) * BY : BX * (BY + 1);  // faces
constexpr int SCRATCH_A = 3 * NSL + 4 * NFC;               // slopes + faces (phases 3-5)
// phase 1-2 staging (see k_step), + the predictor's Manning lambda per owned cell
constexpr int SCRATCH_B = 3 * NSL + 3 * BX * BY + RREG + BX * BY;
#if SWF_STEP_SLIM
constexpr int SCRATCH = SCRATCH_A;  // lambda per owned cell lives in the face planes until phase 3
#else
constexpr int SCRATCH = SCRATCH_A > SCRATCH_B ? SCRATCH_A : SCRATCH_B;
#endif

struct StepArgs {
  const double* __restrict__ H;
  const double* __restrict__ HUx;
  const double* __restrict__ HUy;
  const double* __restrict__ b;
  const double* __restrict__ nf;
  const double* __restrict__ fpx;
  const double* __restrict__ fpy;
  const double* __restrict__ lamn;  // SWF_LAMBDA_SHARE (see ForcesArgs)
  double* __restrict__ gxy;         // SWF_GRAD_SHARE: (gx, gy) per wet owned cell
  double* __restrict__ Ho;
  double* __restrict__ HUxo;
  double* __restrict__ HUyo;
  const DevSrc* src;
  const double* sig;  // [0,nsrc): t_n, [nsrc,2nsrc): t_mid
  const unsigned char* bflag;
  const unsigned char* tile_act;
  unsigned char* tile_same;
  const unsigned* tile_srcm;  // per owned tile: source specs meeting the tile +- 2 cells
  int* redo;                  // tiles whose speculative divisions were rejected
  int* list;                  // work list of k_slist / k_step_list
  FaceTaps taps;              // faces whose tau * fm this step records (nested grids)
  // P2P halo (strips): the neighbours' NEXT-parity state buffers, mapped into
  // this process; owned rows within HALO of a strip edge are also stored
  // there, at the neighbour's local row = ours + peer_drow
  double* peer[2][3];         // [south, north][H, HUx, HUy]
  int peer_drow[2];
  double* hH;                 // pinned host arrays of a host-buffer step (write-through), or null
  double* hHUx;
  double* hHUy;
  double* part;  // 3 per tile
  StepScalars* sc;
  // split step (k_lag -> k_flux): the half-step view of every cell of the
  // flux-active tiles (and of the 2 ghost rows next to a strip's owned rows)
  double* hd;
  double* hu;
  double* hv;
  int* redo_l;  // k_lag tiles to redo exactly
  // exact-diagnostics terms (full grids; null on strips), see swf_ctx
  double* xdef;   // clamp deficit of every flux-on cell of the step
  double* xsrc;   // Ht - Hn of every active cell of the step
  double* xface;  // mass flux of every edge face the step computed
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

// Minmod slopes of one wet cell along one direction.  reconstruct_side
// (stepper.cpp:95-111) computes, for the face on the cell's + side,
// minmod((X[k+1]-X[k])/d_in, (X[k]-X[k-1])/d_out) and for the face on its
// - side the same two quotients negated in numerator and denominator and in
// swapped order; IEEE division is sign-symmetric and minmod is symmetric, so
// both faces use identical slopes and each cell computes them once.
struct Slopes {
  double eta, un, ut;
};

// minmod without branches: for operands of one sign (both > 0 or both < 0)
// the one of smaller magnitude is std::min / std::max of stepper.cpp:23-27
// (equal magnitudes: the same bits); anything else -- mixed signs, zeros,
// NaN -- is 0 as there.
#ifndef SWF_MINMOD_BF
#define SWF_MINMOD_BF 1
#endif
__device__ __forceinline__ double minmod_sel(double a, double b) {
#if SWF_MINMOD_BF
  const bool take = (a > 0.0 && b > 0.0) || (a < 0.0 && b < 0.0);
  const double m = fabs(a) < fabs(b) ? a : b;
  return take ? m : 0.0;
#else
  return minmod(a, b);
#endif
}

__device__ __forceinline__ Slopes cell_slopes(double em, double um, double tm, double sm, double ec,
                                              double uc, double tc, double sc_, double ep, double up,
                                              double tp, double sp, double h, bool* ok = nullptr) {
  // the + side face: in = +1 neighbour, out = -1 neighbour, sgn = +1
  double p_in = 1.0 * h + sp;
  double p_out = -1.0 * h + sm;
  double d_in = p_in - sc_;
  double d_out = sc_ - p_out;
  Slopes s;
  Recip Ri = recip_of(d_in), Ro = recip_of(d_out);
  s.eta = minmod_sel(rdiv(ep - ec, Ri, ok), rdiv(ec - em, Ro, ok));
  s.un = minmod_sel(rdiv(up - uc, Ri, ok), rdiv(uc - um, Ro, ok));
  s.ut = minmod_sel(rdiv(tp - tc, Ri, ok), rdiv(tc - tm, Ro, ok));
  return s;
}

// The P2P halo write of one owned cell: rows within HALO of a strip edge
// also go to the neighbour's ghost rows (same parity, its local row index).
__device__ __forceinline__ void peer_store(const Geo& G, const StepArgs& A, int i, int r,
                                           double h, double qx, double qy) {
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    if (!A.peer[side][0]) continue;
    const bool edge = side == 0 ? r < G.r0 + HALO_ROWS : r >= G.r1 - HALO_ROWS;
    if (!edge) continue;
    const size_t k = (size_t)i + (size_t)(r + A.peer_drow[side]) * G.nx;
    A.peer[side][0][k] = h;
    A.peer[side][1][k] = qx;
    A.peer[side][2][k] = qy;
  }
}

// One side of a face from the cell's slopes (stepper.cpp:112-122).
__device__ __forceinline__ SideState side_from_slopes(double eta, double un, double ut, double sh,
                                                      double b_k, const Slopes& s, double face,
                                                      double b_face) {
  SideState r;
  r.hs = 0.0;
  r.hcell = 0.0;
  r.un = 0.0;
  r.ut = 0.0;
  double off = face - sh;
  double eta_f = eta + s.eta * off;
  r.hcell = smax(0.0, eta_f - b_k);
  if (r.hcell <= 0.0) {
    r.hcell = 0.0;
    return r;
  }
  r.hs = smax(0.0, eta_f - b_face);
  r.un = un + s.un * off;
  r.ut = ut + s.ut * off;
  return r;
}

__device__ __forceinline__ FaceRec face_from_sides(bool wetA, bool wetB, const SideState& L,
                                                   const SideState& R, double g,
                                                   bool* ok = nullptr) {
  FaceRec rec;
  rec.fm = rec.fnl = rec.fnr = rec.ft = 0.0;
  if (!wetA && !wetB) return rec;
  FaceFlux F = hll_face_flux(L.hs, L.un, L.ut, R.hs, R.un, R.ut, g, ok);
  rec.fm = F.fm;
  rec.ft = F.ft;
  rec.fnl = (F.fn - ((0.5 * g) * L.hs) * L.hs) + ((0.5 * g) * L.hcell) * L.hcell;
  rec.fnr = (F.fn - ((0.5 * g) * R.hs) * R.hs) + ((0.5 * g) * R.hcell) * R.hcell;
  return rec;
}

// ---- TMA: the region tiles of k_step (Blackwell tensor-memory copies) -------
// One thread arms an mbarrier with the byte count and issues four 2D tensor
// copies (H, HUx, HUy, b; box = RX x RY doubles, out-of-bounds cells zero-
// filled exactly like the per-thread loads' domain check); every thread
// waits on the barrier's phase.  No registers hold the region in flight.
struct TmaArgs {
  CUtensorMap m[4];  // H, HUx, HUy of the step-start buffer, b
  int on;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void tma_region_loads(const TmaArgs& T, double* R, uint64_t* bar,
                                                 int c0, int c1) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the threads' last smem use
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(4 * RREG * (int)sizeof(double))
               : "memory");
  const int planes[4] = {F_D, F_U, F_V, F_B};
#pragma unroll
  for (int q = 0; q < 4; ++q)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(R + planes[q] * RREG)),
        "l"(reinterpret_cast<uint64_t>(&T.m[q])), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
}

// region-plane accessors of step_tile: eta and the shifts stored, or (slim
// variant) recomputed from depth, bed and velocity with the same expressions
#if SWF_STEP_SLIM
struct SNbrB {  // SNbr with eta = depth + b at the point of use
  bool in;
  const double *d, *b, *u, *v;
  int q;
  __device__ __forceinline__ double dep() const { return d[q]; }
  __device__ __forceinline__ double et() const { return d[q] + b[q]; }
  __device__ __forceinline__ double vx() const { return u[q]; }
  __device__ __forceinline__ double vy() const { return v[q]; }
};
#define R_E(q) (R[F_D * RREG + (q)] + R[F_B * RREG + (q)])
#define R_SX(q) (0.5 * (tau * R[F_U * RREG + (q)]))
#define R_SY(q) (0.5 * (tau * R[F_V * RREG + (q)]))
#define NB_VIEW(in, q) SNbrB{in, R + F_D * RREG, R + F_B * RREG, R + F_U * RREG, R + F_V * RREG, q}
#else
#define R_E(q) R[F_E * RREG + (q)]
#define R_SX(q) R[F_SX * RREG + (q)]
#define R_SY(q) R[F_SY * RREG + (q)]
#define NB_VIEW(in, q) SNbr{in, R + F_D * RREG, R + F_E * RREG, R + F_U * RREG, R + F_V * RREG, q}
#endif

template <bool SPEC>
__device__ __forceinline__ void step_tile(const Geo& G, const StepArgs& A, const int tile,
                                          const TmaArgs& T, uint64_t* mbar, uint32_t& tphase) {
  extern __shared__ __align__(128) double smem[];
  double* R = smem;                       // F_NUM x RREG
  double* SL = smem + F_NUM * RREG;       // 3 x NSL slopes (eta, un, ut)
  double* FB = SL + 3 * NSL;              // 4 x NFC faces (fm, fnl, fnr, ft)
  __shared__ double s_red[3][STHR / 32];
  __shared__ unsigned char s_bf[MAXBF];
  __shared__ unsigned short s_bcol[BX], s_brow[BY];  // B-block column / row of each tile column / row
  __shared__ int s_dflag;  // a clamp deficit in this tile (exact-volume terms to store)
  const PhysConst& P = G.P;  // reciprocals refined at context creation (fused_prepare)
  StepScalars* sc = A.sc;
  if (threadIdx.x == 0) s_dflag = 0;
  // (not stopped(): see StepScalars::step_open)
  if (__syncthreads_or(!*(volatile const int*)&sc->step_open)) return;
  bool sok = true;  // every speculative division of this thread accepted
  unsigned long long my_err = ERR_NONE;  // published once the tile is known exact
  const int tid = threadIdx.x;
  const int tx = tile % G.tiles_x, ty = tile / G.tiles_x;
  const int i0 = tx * BX;         // first owned column
  const int r0 = G.r0 + ty * BY;  // first owned local row
  const size_t nx = G.nx;

  // ---- inactive tile: keep the step-start state (skip semantics) ----------
  if (!(A.tile_act[tile] & 2)) {
    if (!A.tile_same[tile]) {
      for (int c = tid; c < BX * BY; c += STHR) {
        int i = i0 + c % BX, r = r0 + c / BX;
        if (i < G.nx && r < G.r1) {
          size_t k = (size_t)i + (size_t)r * nx;
          A.Ho[k] = A.H[k];
          A.HUxo[k] = A.HUx[k];
          A.HUyo[k] = A.HUy[k];
          peer_store(G, A, i, r, A.H[k], A.HUx[k], A.HUy[k]);
        }
      }
      if (tid == 0) A.tile_same[tile] = 1;
      if (A.peer[0][0] || A.peer[1][0]) __threadfence_system();
    }
    if (tid < 3) A.part[5 * (size_t)tile + tid] = 0.0;
    return;
  }

#ifdef SWF_PHASE_TIMING
  long long t_ph = clock64();
#endif
  // per-tile source masks are precomputed at set_sources (tile +- 2 cells);
  // every per-step scalar is loaded here, ahead of the region loads
  const unsigned srcm = A.tile_srcm[tile];
  const double tau = sc->tau;
  const double half_tau = 0.5 * tau;
  const double wmx = sc->wind_mid[0], wmy = sc->wind_mid[1];
  // the tile's B-block flags (phase 5), staged once
  const int bi_lo = i0 / G.bs, bj_lo = (G.jg0 + r0) / G.bs;
  const int nbi = (min(i0 + BX, G.nx) - 1) / G.bs - bi_lo + 1;
  const int nbj = (min(G.jg0 + r0 + BY, G.jg0 + G.r1) - 1) / G.bs - bj_lo + 1;
  const bool bf_staged = nbi * nbj <= MAXBF;
  if (bf_staged && tid < nbi * nbj)
    s_bf[tid] = A.bflag[(bi_lo + tid % nbi) + (bj_lo + tid / nbi - G.bj0) * G.nbx];
  // the block indices phase 5 needs per cell, one division per column / row
  if (tid >= STHR - BX) s_bcol[tid - (STHR - BX)] = (i0 + tid - (STHR - BX)) / G.bs;
  else if (tid >= STHR - BX - BY) s_brow[tid - (STHR - BX - BY)] = (G.jg0 + r0 + tid - (STHR - BX - BY)) / G.bs;
  const int nsrc = G.nsrc;
  const double* sig_n = A.sig;
  const double* sig_m = A.sig + nsrc;

  // ---- phase 1a: stage the region's inputs in shared memory ----------------
  // All loads of a thread are independent (memory-level parallelism); the
  // slope/face buffers (SL, FB: 3904 doubles) are free until phase 3 and hold
  // f', n and the owned cells' step-start state meanwhile.
  // Phase 2 reads OWN and NF after phase-2 threads may already be writing the
  // x slopes (no barrier between them), so both live above the slope block.
#if SWF_STEP_SLIM
  // lambda(H12, n) of the owned cells as the predictor evaluated it (or -1),
  // in the face planes, which phase 4x writes only after phase 2 is done
  double* LAM = FB;
  static_assert(4 * BX * BY <= 4 * NFC, "lambda plane + the owned step-start state (SWF_OWN_FB)");

  const bool tma = SWF_TMA && T.on;
  if (tma) {  // the region's inputs by TMA into the D, U, V, B planes
    if (tid == 0) tma_region_loads(T, R, mbar, i0 - 2, r0 - 2);
    mbar_wait(mbar, tphase);
    tphase ^= 1u;
  }
  PHASE_MARK(0);
  // ---- phase 1: region inputs and the half-step view (K4 predictor, HalfView)
  // (each thread loads its cells' inputs here: the predictor of a cell needs
  // that cell only, so loads and predictor share one pass and no barrier)
  SWF_PHASE_LOOP
  for (int c = tid; c < RREG; c += STHR) {
    int xr = c % RX, yr = c / RX;
    int i = i0 - 2 + xr, r = r0 - 2 + yr;
    double d = 0.0, u = 0.0, v = 0.0;
    double Hn = 0.0, mx = 0.0, my = 0.0;
    if (tma) {  // (zero outside the local grid, like the loads below)
      Hn = R[F_D * RREG + c];
      mx = R[F_U * RREG + c];
      my = R[F_V * RREG + c];
    } else {
      double bb = 0.0;
      if (i >= 0 && i < G.nx && r >= 0 && r < G.rows) {
        size_t k = (size_t)i + (size_t)r * nx;
        Hn = A.H[k];
        mx = A.HUx[k];
        my = A.HUy[k];
        bb = A.b[k];
      }
      R[F_B * RREG + c] = bb;
    }
    const bool owned = xr >= 2 && xr < BX + 2 && yr >= 2 && yr < BY + 2;
    const int o = (xr - 2) + (yr - 2) * BX;
    if (SWF_OWN_FB && owned) {  // the step-start state, for phase 2 (FB is free until 4x)
      FB[BX * BY + o] = Hn;
      FB[2 * BX * BY + o] = mx;
      FB[3 * BX * BY + o] = my;
    }
    double lam = -1.0;
    if (i >= 0 && i < G.nx && r >= 0 && r < G.rows) {
      const size_t k = (size_t)i + (size_t)r * nx;
      double sg = srcm ? msig(G, A.src, sig_n, srcm, i, G.jg0 + r) : 0.0;
      bool act = Hn > P.eps || sg != 0.0;
      d = Hn;
      Recip Rd{0.0, 0.0};
      if (act) {
        bool wet = Hn > P.eps;
        double fx = wet ? A.fpx[k] : 0.0, fy = wet ? A.fpy[k] : 0.0;
        double Hk = -1.0;
        if (SWF_LAMBDA_SHARE && wet && sg == 0.0) {
          lam = A.lamn[k];
          Hk = Hn;
        }
        predict_cell(Hn, mx, my, sg, fx, fy, G.has_nfield ? A.nf[k] : G.n_manning, half_tau,
                     P.eps, P.g, d, mx, my, SP, &lam, &Rd, Hk);
      }
      if (d > P.eps) {
        u = rdiv(mx, Rd, SP);
        v = rdiv(my, Rd, SP);
      }
    }
    R[F_D * RREG + c] = d;
    R[F_U * RREG + c] = u;
    R[F_V * RREG + c] = v;
    if (owned) LAM[o] = lam;
  }
  __syncthreads();
#else
  double* SC = SL;                      // [0,RREG) fpx  [RREG,2RREG) fpy   (phase 1 only)
  double* OWN = SL + 3 * NSL;           // 3 x (BX*BY): H, HUx, HUy at t_n of owned cells
  double* NF = OWN + 3 * BX * BY;       // RREG: Manning n of the region
  // BX*BY: lambda(H12, n) of owned cells as the predictor evaluated it, or -1
  double* LAM = NF + RREG;
  static_assert(2 * RREG <= 3 * NSL, "phase-1 scratch overlaps OWN");
  static_assert(3 * NSL + 3 * BX * BY + RREG + BX * BY <= SCRATCH,
                "phase-1 scratch overflow");

  for (int c = tid; c < RREG; c += STHR) {
    int i = i0 - 2 + c % RX, r = r0 - 2 + c / RX;
    double h = 0.0, mx = 0.0, my = 0.0, bb = 0.0, fx = 0.0, fy = 0.0, n = G.n_manning;
    double lm = -1.0;
    if (i >= 0 && i < G.nx && r >= 0 && r < G.rows) {
      size_t k = (size_t)i + (size_t)r * nx;
      h = A.H[k];
      mx = A.HUx[k];
      my = A.HUy[k];
      bb = A.b[k];
      fx = A.fpx[k];  // meaningful for wet cells only (k_forces writes those)
      fy = A.fpy[k];
      if (G.has_nfield) n = A.nf[k];
      if (SWF_LAMBDA_SHARE) lm = A.lamn[k];  // likewise
    }
    if (SWF_LAMBDA_SHARE) R[F_SX * RREG + c] = lm;  // the shift plane is free until 1b
    R[F_D * RREG + c] = h;
    R[F_U * RREG + c] = mx;
    R[F_V * RREG + c] = my;
    R[F_B * RREG + c] = bb;
    SC[c] = fx;
    SC[RREG + c] = fy;
    NF[c] = n;
  }
  __syncthreads();

  PHASE_MARK(0);
  // ---- phase 1b: half-step view on the region (K4 predictor, HalfView) -----
  for (int c = tid; c < RREG; c += STHR) {
    int xr = c % RX, yr = c / RX;
    int i = i0 - 2 + xr, r = r0 - 2 + yr;
    double d = 0.0, e = 0.0, u = 0.0, v = 0.0, sx = 0.0, sy = 0.0;
    double Hn = R[F_D * RREG + c], mx = R[F_U * RREG + c], my = R[F_V * RREG + c];
    double bb = R[F_B * RREG + c];
    const bool owned = xr >= 2 && xr < BX + 2 && yr >= 2 && yr < BY + 2;
    const int o = (xr - 2) + (yr - 2) * BX;
    if (owned) {  // keep t_n
      OWN[o] = Hn;
      OWN[BX * BY + o] = mx;
      OWN[2 * BX * BY + o] = my;
    }
    double lam = -1.0;
    if (i >= 0 && i < G.nx && r >= 0 && r < G.rows) {
      double sg = srcm ? msig(G, A.src, sig_n, srcm, i, G.jg0 + r) : 0.0;
      bool act = Hn > P.eps || sg != 0.0;
      d = Hn;
      Recip Rd{0.0, 0.0};
      if (act) {
        bool wet = Hn > P.eps;
        double fx = wet ? SC[c] : 0.0, fy = wet ? SC[RREG + c] : 0.0;
        // without a source H12 == H_n: k_forces' lambda(H_n, n) is lambda(H12, n)
        double Hk = -1.0;
        if (SWF_LAMBDA_SHARE && wet && sg == 0.0) {
          lam = R[F_SX * RREG + c];
          Hk = Hn;
        }
        predict_cell(Hn, mx, my, sg, fx, fy, NF[c], half_tau, P.eps, P.g, d, mx, my, SP, &lam,
                     &Rd, Hk);  // Rd = recip_of(H12) whenever H12 > eps
      }
      e = d + bb;
      if (d > P.eps) {  // implies act (an inactive cell has d = Hn <= eps)
        u = rdiv(mx, Rd, SP);
        v = rdiv(my, Rd, SP);
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
    if (owned) LAM[o] = lam;
  }
  __syncthreads();

#endif  // SWF_STEP_SLIM
  PHASE_MARK(1);
  // ---- phase 2: K5 mid forces + K6 corrector on owned active cells ---------
  constexpr int PER = (BX * BY + STHR - 1) / STHR;  // owned cells per thread (2 at 256)
  // (Ht, Qx, Qy) end up as the final update's base state: the Lagrangian
  // state for active cells, the step-start state otherwise (stepper.cpp:641-651)
#if SWF_P2_ROLLED
  // one copy of the phase's code: the base state goes to the output buffers
  // (phase 5 reads it back and overwrites it; an exact redo re-parks it)
#define PARK(m, h, qx_, qy_)                                   \
  do {                                                         \
    if (i < G.nx && r < G.r1) {                                \
      const size_t kp = (size_t)i + (size_t)r * nx;            \
      A.Ho[kp] = (h);                                          \
      A.HUxo[kp] = (qx_);                                      \
      A.HUyo[kp] = (qy_);                                      \
    }                                                          \
  } while (0)
  double srcvol = 0.0;
#pragma unroll 1
#else
#define PARK(m, h, qx_, qy_) \
  do {                       \
    Ht[m] = (h);             \
    Qx[m] = (qx_);           \
    Qy[m] = (qy_);           \
  } while (0)
  double Ht[PER], Qx[PER], Qy[PER];
  double srcvol = 0.0;
#pragma unroll
#endif
  for (int m = 0; m < PER; ++m) {
    int c = tid + m * STHR;
    if (BX * BY % STHR && c >= BX * BY) break;
    int x = c % BX, y = c / BX;
    int i = i0 + x, r = r0 + y;
#if SWF_STEP_SLIM
    double Hn = 0.0, qxn = 0.0, qyn = 0.0;
    if (SWF_OWN_FB) {
      Hn = FB[BX * BY + c];
      qxn = FB[2 * BX * BY + c];
      qyn = FB[3 * BX * BY + c];
    } else if (i < G.nx && r < G.r1) {
      const size_t k0 = (size_t)i + (size_t)r * nx;
      Hn = A.H[k0];
      qxn = A.HUx[k0];
      qyn = A.HUy[k0];
    }
#else
    double Hn = OWN[c], qxn = OWN[BX * BY + c], qyn = OWN[2 * BX * BY + c];
#endif
    if (i >= G.nx || r >= G.r1) continue;
    int s = (x + 2) + (y + 2) * RX;
    int jg = G.jg0 + r;
    double sgn_ = 0.0, svx = 0.0, svy = 0.0, sgm = 0.0;
    if (srcm) {
      sgn_ = msrc(G, A.src, sig_n, srcm, i, jg, svx, svy);
      sgm = msig(G, A.src, sig_m, srcm, i, jg);
    }
    bool act = Hn > P.eps || sgn_ != 0.0;
    if (!act) {
      PARK(m, Hn, qxn, qyn);  // the step-start state is the base
      continue;
    }
#if SWF_STEP_SLIM
    double n = G.has_nfield ? A.nf[(size_t)i + (size_t)r * nx] : G.n_manning;
#else
    double n = NF[s];
#endif
    double d = R[F_D * RREG + s];  // H12
    double fmx = 0.0, fmy = 0.0;
    // lambda depends on (depth, n) only: the predictor's lambda(H12) serves
    // the mid forces, and the corrector reuses it when Ht == H12 (no source)
    double lam = LAM[c], Hk = -1.0;
    if (d > P.eps) {
      auto nb = [&](bool in, int q) {
        return NB_VIEW(in, q);
      };
      auto W = nb(i > 0, s - 1), E = nb(i + 1 < G.nx, s + 1);
      auto S = nb(jg > 0, s - RX), N = nb(jg + 1 < G.ny, s + RX);
      if (!(lam >= 0.0)) lam = manning_lambda(d, P.g, n);
      Hk = d;
      ForceOut o = cell_forces_lam(d, R[F_U * RREG + s], R[F_V * RREG + s], R_E(s),
                                   W, E, S, N, lam, P, G.nwind > 0, wmx, wmy,
                                   nsrc > 0 ? sgm : 0.0, svx, svy, SP);
      fmx = o.fx - o.frx;
      fmy = o.fy - o.fry;
      if (SWF_GRAD_SHARE) {  // the same half-step view gives phase 5's gradient
        const size_t k2 = 2 * ((size_t)i + (size_t)r * nx);
        A.gxy[k2] = o.gx;
        A.gxy[k2 + 1] = o.gy;
      }
    }
    double ht, qx, qy, sv;
    correct_cell(Hn, qxn, qyn, nsrc > 0, sgm, d, fmx, fmy, n, tau, P.eps, P.g, ht, qx, qy, sv,
                 SP, Hk, &lam);
    srcvol += sv;
    // Ht - Hn (stepper.cpp:353-355) for the exact volumes; nonzero only in
    // tiles near a source spec, and every active cell of those is stored
    if (SWF_XDIAG_SRC && srcm && A.xsrc) A.xsrc[(size_t)i + (size_t)r * nx] = sv;
    // CFL abort (stepper.cpp:378-380, 391-399): dr = tau * u12
    double dx = tau * R[F_U * RREG + s], dy = tau * R[F_V * RREG + s];
    double half_h = 0.5 * P.h;
    if (fabs(dx) >= half_h || fabs(dy) >= half_h) {
      int ib = i / G.bs + (jg / G.bs) * G.nbx;
      unsigned long long local = (unsigned long long)((jg % G.bs) * G.bs + (i % G.bs));
      unsigned long long key = (ERR_CFL << 58) | ((unsigned long long)ib << 24) | local;
      my_err = key < my_err ? key : my_err;
    }
    PARK(m, ht, qx, qy);
  }
#undef PARK

  PHASE_MARK(2);
  // ---- phases 3 and 4, x then y: one copy of the slope and face code -------
  // (the two directions differ only in their index maps and in which
  // velocity is normal; a rolled loop keeps k_step's code -- and its
  // instruction-cache footprint -- to one copy)
  double outflow = 0.0;
  const double face_p = (1.0 * 0.5) * P.h, face_m = (-1.0 * 0.5) * P.h;
  double px_m[PER], px_a[PER], px_c[PER];  // (W.fm-E.fm), (W.fnr-E.fnl), (W.ft-E.ft)
#pragma unroll 1
  for (int dir = 0; dir < 2; ++dir) {
    const double* UN = R + (dir == 0 ? F_U : F_V) * RREG;  // normal velocity
    const double* UT = R + (dir == 0 ? F_V : F_U) * RREG;  // tangential
    const int ds = dir == 0 ? 1 : RX;                        // the next cell along the normal
    // shift along the normal: 0.5*dr (stepper.cpp:72-73)
    auto SH = [&](int q) { return dir == 0 ? R_SX(q) : R_SY(q); };
    // slopes of the cells -1..B of every line of the tile
    const int nsl = dir == 0 ? (BX + 2) * BY : BX * (BY + 2);
    SWF_PHASE_LOOP
    for (int c = tid; c < nsl; c += STHR) {
      int s;
      bool inside;
      if (dir == 0) {
        const int xx = c % (BX + 2), y = c / (BX + 2), i = i0 - 1 + xx;
        s = (xx + 1) + (y + 2) * RX;
        inside = i > 0 && i + 1 < G.nx;
      } else {
        const int x = c % BX, yy = c / BX, jg = G.jg0 + r0 - 1 + yy;
        s = (x + 2) + (yy + 1) * RX;
        inside = jg > 0 && jg + 1 < G.ny && i0 + x < G.nx;
      }
      double se = 0.0, su = 0.0, st = 0.0;
      if (inside && R[F_D * RREG + s] > P.eps) {
        Slopes q = cell_slopes(R_E(s - ds), UN[s - ds], UT[s - ds], SH(s - ds), R_E(s), UN[s],
                               UT[s], SH(s), R_E(s + ds), UN[s + ds], UT[s + ds], SH(s + ds),
                               P.h, SP);
        se = q.eta;
        su = q.un;
        st = q.ut;
      }
      SL[0 * NSL + c] = se;
      SL[1 * NSL + c] = su;
      SL[2 * NSL + c] = st;
    }
    __syncthreads();

    // faces (stepper.cpp:402-494, 496-538)
    const int nfc = dir == 0 ? (BX + 1) * BY : BX * (BY + 1);
    SWF_PHASE_LOOP
    for (int c = tid; c < nfc; c += STHR) {
      // f: the face index along the normal (global), line: the cell line
      // across it (global row of an x face, column of a y face)
      int f, line, sa, la, lb;
      bool valid, edge_lo, edge_hi;
      if (dir == 0) {
        const int fx = c % (BX + 1), y = c / (BX + 1), r = r0 + y;
        f = i0 + fx;
        line = G.jg0 + r;
        valid = f <= G.nx && r < G.r1;
        edge_lo = f == 0;
        edge_hi = f == G.nx;
        sa = (fx + 1) + (y + 2) * RX;  // cell f-1
        la = fx + y * (BX + 2);        // slope slots of cells f-1, f
        lb = la + 1;
      } else {
        const int x = c % BX, fy = c / BX, rf = r0 + fy;
        f = G.jg0 + rf;
        line = i0 + x;
        valid = line < G.nx && rf <= G.r1;
        edge_lo = f == 0;
        edge_hi = f == G.ny;
        sa = (x + 2) + (fy + 1) * RX;  // cell rf-1
        la = x + fy * BX;              // slope slots of rows rf-1, rf
        lb = la + BX;
      }
      FaceRec rec;
      rec.fm = rec.fnl = rec.fnr = rec.ft = 0.0;
      if (valid) {
        if (edge_lo || edge_hi) {
          const bool lo = edge_lo;
          const int se = lo ? sa + ds : sa;
          const double H = R[F_D * RREG + se];
          const bool refl = dir == 0 ? (lo ? G.west_refl : G.east_refl)
                                     : (lo ? G.south_refl : G.north_refl);
          rec = boundary_face(H > P.eps, H, UN[se], UT[se], lo, refl, P.g);
          outflow += lo ? -rec.fm : rec.fm;
          if (A.xface)  // the edge faces in the exact-volume order (W, E by row; S, N by column)
            A.xface[(dir == 0 ? 0 : 2 * G.ny) + (lo ? 0 : (dir == 0 ? G.ny : G.nx)) + line] =
                rec.fm;
        } else {
          const int sb = sa + ds;
          double dA = R[F_D * RREG + sa], dB = R[F_D * RREG + sb];
          bool wetA = dA > P.eps, wetB = dB > P.eps;
          if (wetA || wetB) {
            double bA = R[F_B * RREG + sa], bB = R[F_B * RREG + sb];
            double bf = smax(bA, bB);
            SideState L, Rr;
            L.hs = L.hcell = L.un = L.ut = 0.0;
            Rr = L;
            if (wetA) {
              Slopes q = {SL[la], SL[NSL + la], SL[2 * NSL + la]};
              L = side_from_slopes(R_E(sa), UN[sa], UT[sa], SH(sa), bA, q, face_p, bf);
            }
            if (wetB) {
              Slopes q = {SL[lb], SL[NSL + lb], SL[2 * NSL + lb]};
              Rr = side_from_slopes(R_E(sb), UN[sb], UT[sb], SH(sb), bB, q, face_m, bf);
            }
            rec = face_from_sides(wetA, wetB, L, Rr, P.g, SP);
            if (!face_finite(rec)) {
              unsigned long long key = fused_flux_key(G, A.bflag, dir, line, f);
              my_err = key < my_err ? key : my_err;
            }
          }
        }
      }
      FB[0 * NFC + c] = rec.fm;
      FB[1 * NFC + c] = rec.fnl;
      FB[2 * NFC + c] = rec.fnr;
      FB[3 * NFC + c] = rec.ft;
    }
    __syncthreads();
    // face taps (nested-grid flux correction): each tile records its west /
    // south faces only, so every face is written once; faces no active tile
    // computes stay 0 (dry)
    if (A.taps.n) {
      for (int c = tid; c < nfc; c += STHR) {
        if (dir == 0) {
          const int fx = c % (BX + 1), y = c / (BX + 1), f = i0 + fx, jg = G.jg0 + r0 + y;
          for (int q = 0; q < A.taps.n; ++q)
            if (fx < BX && r0 + y < G.r1 &&
                (f == A.taps.i0[q] || f == A.taps.i0[q] + A.taps.ni[q]) &&
                jg >= A.taps.j0[q] && jg < A.taps.j0[q] + A.taps.nj[q])
              A.taps.out[q][(f == A.taps.i0[q] ? 0 : A.taps.nj[q]) + (jg - A.taps.j0[q])] =
                  tau * FB[0 * NFC + c];
        } else {
          const int x = c % BX, fy = c / BX, i = i0 + x, rf = r0 + fy, jf = G.jg0 + rf;
          for (int q = 0; q < A.taps.n; ++q)
            if (fy < BY && i < G.nx && rf < G.r1 &&
                (jf == A.taps.j0[q] || jf == A.taps.j0[q] + A.taps.nj[q]) &&
                i >= A.taps.i0[q] && i < A.taps.i0[q] + A.taps.ni[q])
              A.taps.out[q][2 * A.taps.nj[q] + (jf == A.taps.j0[q] ? 0 : A.taps.ni[q]) +
                            (i - A.taps.i0[q])] = tau * FB[0 * NFC + c];
        }
      }
    }
    if (dir == 0) {  // the x faces' contributions, before the y faces take the planes
#pragma unroll
      for (int m = 0; m < PER; ++m) {
        int c = tid + m * STHR;
        if (BX * BY % STHR && c >= BX * BY) break;
        int x = c % BX, y = c / BX;
        int w = x + y * (BX + 1), e = w + 1;
        px_m[m] = FB[0 * NFC + w] - FB[0 * NFC + e];
        px_a[m] = FB[2 * NFC + w] - FB[1 * NFC + e];
        px_c[m] = FB[3 * NFC + w] - FB[3 * NFC + e];
      }
      // (the y slopes write only SL; FB is rewritten after the next barrier)
    }
  }
  PHASE_MARK(6);
  // ---- phase 5: accumulate (stepper.cpp:540-566) + final (628-659) ---------
  double deficit = 0.0;
  int hw = 0;  // doubles this thread wrote back to the caller's arrays
  double dfm[PER];  // the clamp deficit of each of the thread's cells (0 if not flux-on)
  const double dt_h = tau / P.h;
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    dfm[m] = 0.0;
    int c = tid + m * STHR;
    if (BX * BY % STHR && c >= BX * BY) break;
    int x = c % BX, y = c / BX;
    int i = i0 + x, r = r0 + y;
    if (i >= G.nx || r >= G.r1) continue;
    int jg = G.jg0 + r;
    int s = (x + 2) + (y + 2) * RX;
    size_t k = (size_t)i + (size_t)r * nx;
    const int bc = s_bcol[x], br = s_brow[y];  // i / bs, jg / bs
    unsigned char bfl = bf_staged ? s_bf[(bc - bi_lo) + (br - bj_lo) * nbi]
                                  : A.bflag[bc + (br - G.bj0) * G.nbx];
    bool flux_on = !G.skip || (bfl & 2);
#if SWF_P2_ROLLED
    const double Htm = A.Ho[k], Qxm = A.HUxo[k], Qym = A.HUyo[k];  // parked in phase 2
#else
    const double Htm = Ht[m], Qxm = Qx[m], Qym = Qy[m];
#endif
    if (!flux_on) {  // block skipped by the reference: state unchanged
      A.Ho[k] = Htm;  // no active cell in such a block: (Ht, Qx, Qy) = step-start state
      A.HUxo[k] = Qxm;
      A.HUyo[k] = Qym;
      peer_store(G, A, i, r, Htm, Qxm, Qym);
      continue;
    }
    int sf = x + y * BX, nf_ = sf + BX;  // S and N face of the cell
    double py_m = FB[0 * NFC + sf] - FB[0 * NFC + nf_];
    double py_a = FB[2 * NFC + sf] - FB[1 * NFC + nf_];  // S.fnr - N.fnl
    double py_c = FB[3 * NFC + sf] - FB[3 * NFC + nf_];  // S.ft - N.ft
    double d = R[F_D * RREG + s];
    bool wet = d > P.eps;
    double cx = 0.0, cy = 0.0;
    if (wet) {
      auto nb = [&](bool in, int q) {
        return NB_VIEW(in, q);
      };
      double gx, gy;
      if (SWF_GRAD_SHARE) {  // phase 2's mid forces computed it for this wet cell
        gx = A.gxy[2 * k];
        gy = A.gxy[2 * k + 1];
      } else {
        double eta_c = R_E(s);
        gx = eta_grad_comp(nb(i > 0, s - 1), nb(i + 1 < G.nx, s + 1), eta_c, P, SP);
        gy = eta_grad_comp(nb(jg > 0, s - RX), nb(jg + 1 < G.ny, s + RX), eta_c, P, SP);
      }
      double gh = (P.g * d) * P.h;
      cx = gh * gx;
      cy = gh * gy;
    }
    double Fh = px_m[m] + py_m;
    double Fvx = (px_a[m] + py_c) + cx;
    double Fvy = (py_a + px_c[m]) + cy;
    double H1, qx, qy, dfc;
    final_cell(Htm, Qxm, Qym, Fh, Fvx, Fvy, dt_h, P.eps, H1, qx, qy, dfc);
    deficit += dfc;
    dfm[m] = dfc;
    A.Ho[k] = H1;
    A.HUxo[k] = qx;
    A.HUyo[k] = qy;
    if (A.hH) {  // host-buffer step: write the updated cell straight into the caller's arrays
      // (every updated cell: skipping the unchanged ones measured slower --
      // 5 % fewer bytes in gappy PCIe writes, profiles/README.md round 3)
      A.hH[k] = H1;
      A.hHUx[k] = qx;
      A.hHUy[k] = qy;
      hw += 3;
    }
    peer_store(G, A, i, r, H1, qx, qy);
  }
  if (tid == 0) A.tile_same[tile] = 0;
  // the neighbour reads these rows after a stream-ordered token from us:
  // make the peer stores visible system-wide before this kernel completes
  if (A.peer[0][0] || A.peer[1][0]) __threadfence_system();

  PHASE_MARK(7);
  if (A.hH) {  // the host-buffer step's write-back volume (one atomic per warp)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hw += __shfl_xor_sync(0xffffffffu, hw, o);
    if ((tid & 31) == 0 && hw) atomicAdd(&sc->host_writes, (unsigned long long)hw);
  }
  // ---- per-tile diagnostic partials (deterministic) ------------------------
  if (deficit != 0.0) s_dflag = 1;  // read after the barriers below
  double v3[3] = {deficit, srcvol, outflow};
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    double v = v3[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) s_red[q][tid >> 5] = v;
  }
#if !SWF_EPI_ONEBAR
  __syncthreads();
  if (tid < 3) {
    double v = 0.0;
    for (int w = 0; w < STHR / 32; ++w) v += s_red[tid][w];
    A.part[5 * (size_t)tile + tid] = v;
  }
#endif
  // a tile with a rejected speculative division is redone exactly (its
  // outputs and partials are overwritten there); otherwise publish errors
  const bool any_bad = __syncthreads_or(!sok);
#if SWF_EPI_ONEBAR
  if (tid < 3) {  // (the barrier above also orders the s_red writes)
    double v = 0.0;
    for (int w = 0; w < STHR / 32; ++w) v += s_red[tid][w];
    A.part[5 * (size_t)tile + tid] = v;
  }
#endif
  const bool redo = SPEC && any_bad;
  if (redo) {
    if (tid == 0) A.redo[atomicAdd(&sc->redo_n[1], 1)] = tile;
  } else {
    if (my_err != ERR_NONE) atomicMin(&sc->err_key, my_err);
    // exact volumes: a tile with a clamp deficit stores every cell's term
    // (the reduction reads the cells of tiles with a nonzero deficit partial)
    if (SWF_XDIAG_DEF && s_dflag && A.xdef) {
#pragma unroll
      for (int m = 0; m < PER; ++m) {
        const int c = tid + m * STHR;
        if (BX * BY % STHR && c >= BX * BY) break;
        const int i = i0 + c % BX, r = r0 + c / BX;
        if (i < G.nx && r < G.r1) A.xdef[(size_t)i + (size_t)r * nx] = dfm[m];
      }
    }
  }
}

__device__ __forceinline__ void step_kernel_init(const TmaArgs& T, uint64_t* mbar) {
  if (SWF_TMA && T.on && threadIdx.x == 0) mbar_init(mbar);
  __syncthreads();
}

__global__ void __launch_bounds__(STHR, SWF_STEP_MINB)
    k_step(Geo G, StepArgs A, const __grid_constant__ TmaArgs T) {
  __shared__ __align__(8) uint64_t s_mbar;
  uint32_t tphase = 0;
  step_kernel_init(T, &s_mbar);
  step_tile<SWF_SPECULATE != 0>(G, A, blockIdx.x, T, &s_mbar, tphase);
}

// k_slist: the tiles k_step must visit -- flux-active ones, and inactive
// ones whose two ping-pong copies still differ; every other tile keeps its
// state and gets zero diagnostics partials here.
__global__ void k_slist(Geo G, StepArgs A) {
  if (stopped(A.sc)) return;  // (see k_flist)
  const int nt = G.tiles_x * G.tiles_y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = t < nt;  // every lane reaches the warp-wide append
  const bool need = valid && ((A.tile_act[t] & 2) || !A.tile_same[t]);
  append_ordered(A.list, &A.sc->list_n[1], need, t);
  if (valid && !need) {
    A.part[5 * (size_t)t + 0] = 0.0;
    A.part[5 * (size_t)t + 1] = 0.0;
    A.part[5 * (size_t)t + 2] = 0.0;
  }
}

__global__ void __launch_bounds__(STHR, SWF_STEP_MINB)
    k_step_list(Geo G, StepArgs A, const __grid_constant__ TmaArgs T) {
  __shared__ int s_next;
  __shared__ __align__(8) uint64_t s_mbar;
  uint32_t tphase = 0;
  step_kernel_init(T, &s_mbar);
  StepScalars* sc = A.sc;
  const int n = *(volatile int*)&sc->list_n[1];
  while (true) {
    if (threadIdx.x == 0) s_next = atomicAdd(&sc->list_take[1], 1);
    __syncthreads();
    const int q = s_next;
    __syncthreads();
    if (q >= n) break;
    step_tile<SWF_SPECULATE != 0>(G, A, A.list[q], T, &s_mbar, tphase);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(STHR, SWF_STEP_MINB)
    k_step_redo(Geo G, StepArgs A, const __grid_constant__ TmaArgs T) {
  __shared__ __align__(8) uint64_t s_mbar;
  uint32_t tphase = 0;
  step_kernel_init(T, &s_mbar);
  const int n = *(volatile int*)&A.sc->redo_n[1];
  for (int q = blockIdx.x; q < n; q += gridDim.x) {
    step_tile<false>(G, A, A.redo[q], T, &s_mbar, tphase);
    __syncthreads();
  }
}


#if !SWF_STEP_SLIM  // the split kernels use the full region planes
// ===========================================================================
// Split step (-DSWF_SPLIT=1; measured and NOT the default): k_step's work in
// two tile kernels, each with its own register and shared-memory budget (the
// fused k_step runs at both limits, 80 registers x 768 threads and 3 x 76 KB
// per SM).  On C3 it is bit-identical but slower: k_lag 5.45 + k_flux 7.26 ms
// against k_step 11.0 ms (profiles/README.md, round 3) -- both halves still
// sit at 24 warps per SM (k_lag's mid forces need 80 registers, k_flux 76)
// while the hand-off adds ~110 B per active cell of HBM traffic and a load
// phase of its own.
//   k_lag  (K4 predictor on the tile + 1-cell halo, K5 mid forces and K6
//          corrector on owned cells): writes the Lagrangian state (Ht, HVt)
//          of every owned cell into the next-parity buffers -- the final
//          update's base state -- and the half-step view (depth, u, v) of
//          every owned cell into d_half.
//   k_ghost_half  the half-step view of the 2 ghost rows next to a strip's
//          owned rows (their predictor; no tile there).
//   k_flux (K7 slopes and faces, K8 final update on owned cells): reads the
//          half-step view on the tile + 2-cell halo and the base state.
// A cell of a tile k_lag did not visit (not flux-active) is not active
// (dry, no source), so its half-step view is its state: (H, 0, 0).
// Same arithmetic, same order as step_tile: bit-identical results.
// ===========================================================================
#ifndef SWF_LAG_THREADS
#define SWF_LAG_THREADS 256
#endif
#ifndef SWF_LAG_MINB
#define SWF_LAG_MINB 3
#endif
#ifndef SWF_FLUX_THREADS
#define SWF_FLUX_THREADS 256
#endif
#ifndef SWF_FLUX_MINB
#define SWF_FLUX_MINB 3
#endif
constexpr int LTHR = SWF_LAG_THREADS, XTHR = SWF_FLUX_THREADS;
static_assert(LTHR % 32 == 0 && XTHR % 32 == 0, "whole warps");
// k_lag shared memory (doubles): 7 region planes (H->D, HUx->U, HUy->V, b->E,
// f'x, f'y, n), then the owned cells' step-start state and lambda(H12)
enum { L_D = 0, L_U, L_V, L_E, L_FX, L_FY, L_N, L_NUM };
constexpr size_t lag_smem() { return (size_t)(L_NUM * AREG + 4 * BX * BY) * sizeof(double); }
// k_flux shared memory: the 2-halo region planes, then slopes and faces
constexpr size_t flux_smem() { return (size_t)(F_NUM * RREG + SCRATCH_A) * sizeof(double); }
static_assert(3 * BX * BY <= 3 * NSL, "k_flux stages its results in the slope planes");

template <bool SPEC>
__device__ __forceinline__ void lag_tile(const Geo& G, const StepArgs& A, const int tile) {
  extern __shared__ double smem[];
  double* Q = smem;                         // L_NUM x AREG
  double* OWN = smem + L_NUM * AREG;        // 3 x (BX*BY): H, HUx, HUy at t_n
  double* LAM = OWN + 3 * BX * BY;          // BX*BY: lambda(H12, n) of the predictor, or -1
  __shared__ double s_red[LTHR / 32];
  const PhysConst& P = G.P;
  StepScalars* sc = A.sc;
  if (__syncthreads_or(stopped(sc))) return;
  if (!(A.tile_act[tile] & 2)) return;  // k_flux keeps the state of an inactive tile
  bool sok = true;
  unsigned long long my_err = ERR_NONE;
  const int tid = threadIdx.x;
  const int tx = tile % G.tiles_x, ty = tile / G.tiles_x;
  const int i0 = tx * BX;
  const int r0 = G.r0 + ty * BY;
  const size_t nx = G.nx;
  const unsigned srcm = A.tile_srcm[tile];  // specs meeting the tile +- 2 cells
  const double tau = sc->tau;
  const double half_tau = 0.5 * tau;
  const double wmx = sc->wind_mid[0], wmy = sc->wind_mid[1];
  const int nsrc = G.nsrc;
  const double* sig_n = A.sig;
  const double* sig_m = A.sig + nsrc;

  // ---- L1a: stage the region's inputs (tile + 1-cell halo) ----------------
  for (int c = tid; c < AREG; c += LTHR) {
    int i = i0 - 1 + c % AREGX, r = r0 - 1 + c / AREGX;
    double h = 0.0, mx = 0.0, my = 0.0, bb = 0.0, fx = 0.0, fy = 0.0, n = G.n_manning;
    if (i >= 0 && i < G.nx && r >= 0 && r < G.rows) {
      size_t k = (size_t)i + (size_t)r * nx;
      h = A.H[k];
      mx = A.HUx[k];
      my = A.HUy[k];
      bb = A.b[k];
      fx = A.fpx[k];
      fy = A.fpy[k];
      if (G.has_nfield) n = A.nf[k];
    }
    Q[L_D * AREG + c] = h;
    Q[L_U * AREG + c] = mx;
    Q[L_V * AREG + c] = my;
    Q[L_E * AREG + c] = bb;
    Q[L_FX * AREG + c] = fx;
    Q[L_FY * AREG + c] = fy;
    Q[L_N * AREG + c] = n;
  }
  __syncthreads();

  // ---- L1b: K4 predictor -> half-step view (in place) ----------------------
  for (int c = tid; c < AREG; c += LTHR) {
    int xr = c % AREGX, yr = c / AREGX;
    int i = i0 - 1 + xr, r = r0 - 1 + yr;
    double Hn = Q[L_D * AREG + c], mx = Q[L_U * AREG + c], my = Q[L_V * AREG + c];
    double bb = Q[L_E * AREG + c];
    double d = 0.0, u = 0.0, v = 0.0;
    const bool owned = xr >= 1 && xr < BX + 1 && yr >= 1 && yr < BY + 1;
    const int o = (xr - 1) + (yr - 1) * BX;
    if (owned) {
      OWN[o] = Hn;
      OWN[BX * BY + o] = mx;
      OWN[2 * BX * BY + o] = my;
    }
    double lam = -1.0;
    const bool in = i >= 0 && i < G.nx && r >= 0 && r < G.rows;
    if (in) {
      double sg = srcm ? msig(G, A.src, sig_n, srcm, i, G.jg0 + r) : 0.0;
      bool act = Hn > P.eps || sg != 0.0;
      d = Hn;
      Recip Rd{0.0, 0.0};
      if (act) {
        bool wet = Hn > P.eps;
        double fx = wet ? Q[L_FX * AREG + c] : 0.0, fy = wet ? Q[L_FY * AREG + c] : 0.0;
        predict_cell(Hn, mx, my, sg, fx, fy, Q[L_N * AREG + c], half_tau, P.eps, P.g, d, mx, my,
                     SP, &lam, &Rd);
      }
      if (d > P.eps) {
        u = rdiv(mx, Rd, SP);
        v = rdiv(my, Rd, SP);
      }
    }
    Q[L_D * AREG + c] = d;
    Q[L_E * AREG + c] = d + bb;
    Q[L_U * AREG + c] = u;
    Q[L_V * AREG + c] = v;
    if (owned) {
      LAM[o] = lam;
      if (i < G.nx && r < G.r1) {  // the half-step view for k_flux
        size_t k = (size_t)i + (size_t)r * nx;
        A.hd[k] = d;
        A.hu[k] = u;
        A.hv[k] = v;
      }
    }
  }
  __syncthreads();

  // ---- L2: K5 mid forces + K6 corrector on owned cells ---------------------
  double srcvol = 0.0;
  const double* QD = Q + L_D * AREG;
  const double* QE = Q + L_E * AREG;
  const double* QU = Q + L_U * AREG;
  const double* QV = Q + L_V * AREG;
  for (int c = tid; c < BX * BY; c += LTHR) {
    int x = c % BX, y = c / BX;
    int i = i0 + x, r = r0 + y;
    if (i >= G.nx || r >= G.r1) continue;
    const size_t k = (size_t)i + (size_t)r * nx;
    double Hn = OWN[c], qxn = OWN[BX * BY + c], qyn = OWN[2 * BX * BY + c];
    int s = (x + 1) + (y + 1) * AREGX;
    int jg = G.jg0 + r;
    double sgn_ = 0.0, svx = 0.0, svy = 0.0, sgm = 0.0;
    if (srcm) {
      sgn_ = msrc(G, A.src, sig_n, srcm, i, jg, svx, svy);
      sgm = msig(G, A.src, sig_m, srcm, i, jg);
    }
    bool act = Hn > P.eps || sgn_ != 0.0;
    double ht = Hn, qx = qxn, qy = qyn;  // base state of an inactive cell (stepper.cpp:641-651)
    if (act) {
      double n = Q[L_N * AREG + s];
      double d = QD[s];  // H12
      double fmx = 0.0, fmy = 0.0;
      double lam = LAM[c], Hk = -1.0;
      if (d > P.eps) {
        auto nb = [&](bool inb, int q) { return SNbr{inb, QD, QE, QU, QV, q}; };
        SNbr W = nb(i > 0, s - 1), E = nb(i + 1 < G.nx, s + 1);
        SNbr S = nb(jg > 0, s - AREGX), N = nb(jg + 1 < G.ny, s + AREGX);
        if (!(lam >= 0.0)) lam = manning_lambda(d, P.g, n);
        Hk = d;
        ForceOut o = cell_forces_lam(d, QU[s], QV[s], QE[s], W, E, S, N, lam, P, G.nwind > 0, wmx,
                                     wmy, nsrc > 0 ? sgm : 0.0, svx, svy, SP);
        fmx = o.fx - o.frx;
        fmy = o.fy - o.fry;
      }
      double sv;
      correct_cell(Hn, qxn, qyn, nsrc > 0, sgm, d, fmx, fmy, n, tau, P.eps, P.g, ht, qx, qy, sv,
                   SP, Hk, &lam);
      srcvol += sv;
      double dx = tau * QU[s], dy = tau * QV[s];
      double half_h = 0.5 * P.h;
      if (fabs(dx) >= half_h || fabs(dy) >= half_h) {
        int ib = i / G.bs + (jg / G.bs) * G.nbx;
        unsigned long long local = (unsigned long long)((jg % G.bs) * G.bs + (i % G.bs));
        unsigned long long key = (ERR_CFL << 58) | ((unsigned long long)ib << 24) | local;
        my_err = key < my_err ? key : my_err;
      }
    }
    A.Ho[k] = ht;  // the final update's base state (k_flux reads it back)
    A.HUxo[k] = qx;
    A.HUyo[k] = qy;
  }

  // ---- the tile's source-volume partial (deterministic) --------------------
  double v = srcvol;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((tid & 31) == 0) s_red[tid >> 5] = v;
  const bool any_bad = __syncthreads_or(!sok);
  if (tid == 0) {
    double w = 0.0;
    for (int q = 0; q < LTHR / 32; ++q) w += s_red[q];
    A.part[5 * (size_t)tile + 1] = w;
  }
  if (SPEC && any_bad) {
    if (tid == 0) A.redo_l[atomicAdd(&sc->redo_n[2], 1)] = tile;
  } else if (my_err != ERR_NONE) {
    atomicMin(&sc->err_key, my_err);
  }
}

__global__ void __launch_bounds__(LTHR, SWF_LAG_MINB) k_lag_list(Geo G, StepArgs A) {
  __shared__ int s_next;
  StepScalars* sc = A.sc;
  const int n = *(volatile int*)&sc->list_n[1];
  while (true) {
    if (threadIdx.x == 0) s_next = atomicAdd(&sc->list_take[2], 1);
    __syncthreads();
    const int q = s_next;
    __syncthreads();
    if (q >= n) break;
    lag_tile<SWF_SPECULATE != 0>(G, A, A.list[q]);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(LTHR, SWF_LAG_MINB) k_lag_redo(Geo G, StepArgs A) {
  const int n = *(volatile int*)&A.sc->redo_n[2];
  for (int q = blockIdx.x; q < n; q += gridDim.x) {
    lag_tile<false>(G, A, A.redo_l[q]);
    __syncthreads();
  }
}

// The half-step view of the ghost rows k_flux reads next to a strip's owned
// rows (local rows [r0-2, r0) and [r1, r1+2)): one thread per cell, the
// predictor exactly (stepper.cpp:269-308; f' is valid there, k_forces covers
// 2 ghost rows).
__global__ void k_ghost_half(Geo G, StepArgs A) {
  const StepScalars* sc = A.sc;
  if (stopped(sc)) return;
  const PhysConst& P = G.P;
  const int lo = G.r0 >= 2 ? 2 : G.r0;                 // ghost rows below
  const int hi = G.rows - G.r1 >= 2 ? 2 : G.rows - G.r1;  // and above
  const int nrow = lo + hi;
  const size_t total = (size_t)nrow * G.nx;
  const double half_tau = 0.5 * sc->tau;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const int q = (int)(t / G.nx), i = (int)(t % G.nx);
    const int r = q < lo ? G.r0 - lo + q : G.r1 + (q - lo);
    const size_t k = (size_t)i + (size_t)r * G.nx;
    const double Hn = A.H[k];
    double mx = A.HUx[k], my = A.HUy[k];
    const double sg = G.nsrc > 0 ? cell_sigma_only(A.src, A.sig, G.nsrc, i, G.jg0 + r) : 0.0;
    const bool act = Hn > P.eps || sg != 0.0;
    double d = Hn, u = 0.0, v = 0.0;
    Recip Rd{0.0, 0.0};
    if (act) {
      const bool wet = Hn > P.eps;
      predict_cell(Hn, mx, my, sg, wet ? A.fpx[k] : 0.0, wet ? A.fpy[k] : 0.0,
                   G.has_nfield ? A.nf[k] : G.n_manning, half_tau, P.eps, P.g, d, mx, my,
                   nullptr, nullptr, &Rd);
    }
    if (d > P.eps) {
      u = rdiv(mx, Rd);
      v = rdiv(my, Rd);
    }
    A.hd[k] = d;
    A.hu[k] = u;
    A.hv[k] = v;
  }
}

template <bool SPEC>
__device__ __forceinline__ void flux_tile(const Geo& G, const StepArgs& A, const int tile) {
  extern __shared__ double smem[];
  double* R = smem;                  // F_NUM x RREG
  double* SL = smem + F_NUM * RREG;  // 3 x NSL slopes (eta, un, ut)
  double* FB = SL + 3 * NSL;         // 4 x NFC faces (fm, fnl, fnr, ft)
  __shared__ double s_red[2][XTHR / 32];
  __shared__ unsigned char s_bf[MAXBF];
  __shared__ unsigned short s_bcol[BX], s_brow[BY];
  __shared__ unsigned char s_nact[9];  // flux-active flags of the 3 x 3 tiles around
  const PhysConst& P = G.P;
  StepScalars* sc = A.sc;
  if (__syncthreads_or(stopped(sc))) return;
  bool sok = true;
  unsigned long long my_err = ERR_NONE;
  const int tid = threadIdx.x;
  const int tx = tile % G.tiles_x, ty = tile / G.tiles_x;
  const int i0 = tx * BX;
  const int r0 = G.r0 + ty * BY;
  const size_t nx = G.nx;

  // ---- inactive tile: keep the step-start state (skip semantics) ----------
  if (!(A.tile_act[tile] & 2)) {
    if (!A.tile_same[tile]) {
      for (int c = tid; c < BX * BY; c += XTHR) {
        int i = i0 + c % BX, r = r0 + c / BX;
        if (i < G.nx && r < G.r1) {
          size_t k = (size_t)i + (size_t)r * nx;
          A.Ho[k] = A.H[k];
          A.HUxo[k] = A.HUx[k];
          A.HUyo[k] = A.HUy[k];
          peer_store(G, A, i, r, A.H[k], A.HUx[k], A.HUy[k]);
        }
      }
      if (tid == 0) A.tile_same[tile] = 1;
      if (A.peer[0][0] || A.peer[1][0]) __threadfence_system();
    }
    if (tid < 3) A.part[5 * (size_t)tile + tid] = 0.0;
    return;
  }

  const double tau = sc->tau;
  const int bi_lo = i0 / G.bs, bj_lo = (G.jg0 + r0) / G.bs;
  const int nbi = (min(i0 + BX, G.nx) - 1) / G.bs - bi_lo + 1;
  const int nbj = (min(G.jg0 + r0 + BY, G.jg0 + G.r1) - 1) / G.bs - bj_lo + 1;
  const bool bf_staged = nbi * nbj <= MAXBF;
  if (bf_staged && tid < nbi * nbj)
    s_bf[tid] = A.bflag[(bi_lo + tid % nbi) + (bj_lo + tid / nbi - G.bj0) * G.nbx];
  if (tid >= XTHR - BX) s_bcol[tid - (XTHR - BX)] = (i0 + tid - (XTHR - BX)) / G.bs;
  else if (tid >= XTHR - BX - BY) s_brow[tid - (XTHR - BX - BY)] = (G.jg0 + r0 + tid - (XTHR - BX - BY)) / G.bs;
  else if (tid < 9) {
    const int ntx = tx + tid % 3 - 1, nty = ty + tid / 3 - 1;
    // outside the owned tile rows: ghost rows (k_ghost_half) count as visited
    s_nact[tid] = (ntx < 0 || ntx >= G.tiles_x) ? 0
                  : (nty < 0 || nty >= G.tiles_y) ? 1
                  : ((A.tile_act[ntx + nty * G.tiles_x] & 2) != 0);
  }
  __syncthreads();

  // ---- F1: the half-step view on the region (tile + 2-cell halo) ----------
  for (int c = tid; c < RREG; c += XTHR) {
    const int xr = c % RX, yr = c / RX;
    const int i = i0 - 2 + xr, r = r0 - 2 + yr;
    double d = 0.0, e = 0.0, u = 0.0, v = 0.0, sx = 0.0, sy = 0.0, bb = 0.0;
    if (i >= 0 && i < G.nx && r >= 0 && r < G.rows) {
      const size_t k = (size_t)i + (size_t)r * nx;
      const int gx = xr < 2 ? 0 : (xr < BX + 2 ? 1 : 2);
      const int gy = yr < 2 ? 0 : (yr < BY + 2 ? 1 : 2);
      const bool ghost = r < G.r0 || r >= G.r1;
      bb = A.b[k];
      if (ghost || s_nact[gx + 3 * gy]) {
        d = A.hd[k];
        u = A.hu[k];
        v = A.hv[k];
      } else {
        d = A.H[k];  // not active: the state itself, at rest
      }
      e = d + bb;
      // shift = 0.5*dr, dr = tau*u12 (stepper.cpp:72-73, 373-379); 0 for an
      // inactive cell, whose u is 0
      sx = 0.5 * (tau * u);
      sy = 0.5 * (tau * v);
    }
    R[F_D * RREG + c] = d;
    R[F_E * RREG + c] = e;
    R[F_U * RREG + c] = u;
    R[F_V * RREG + c] = v;
    R[F_SX * RREG + c] = sx;
    R[F_SY * RREG + c] = sy;
    R[F_B * RREG + c] = bb;
  }
  __syncthreads();
    constexpr int PER = (BX * BY + XTHR - 1) / XTHR;  // owned cells per thread
  // ---- phase 3x: x slopes of columns -1..BX (rows of the tile) -------------
  for (int c = tid; c < (BX + 2) * BY; c += XTHR) {
    int xx = c % (BX + 2), y = c / (BX + 2);
    int i = i0 - 1 + xx;
    int s = (xx + 1) + (y + 2) * RX;
    double se = 0.0, su = 0.0, st = 0.0;
    if (i > 0 && i + 1 < G.nx && R[F_D * RREG + s] > P.eps) {
      Slopes q = cell_slopes(R[F_E * RREG + s - 1], R[F_U * RREG + s - 1], R[F_V * RREG + s - 1],
                             R[F_SX * RREG + s - 1], R[F_E * RREG + s], R[F_U * RREG + s],
                             R[F_V * RREG + s], R[F_SX * RREG + s], R[F_E * RREG + s + 1],
                             R[F_U * RREG + s + 1], R[F_V * RREG + s + 1], R[F_SX * RREG + s + 1],
                             P.h, SP);
      se = q.eta;
      su = q.un;
      st = q.ut;
    }
    SL[0 * NSL + c] = se;
    SL[1 * NSL + c] = su;
    SL[2 * NSL + c] = st;
  }
  __syncthreads();

  // ---- phase 4x: x faces (stepper.cpp:402-447, 496-516) ----------------------
  double outflow = 0.0;
  const double face_p = (1.0 * 0.5) * P.h, face_m = (-1.0 * 0.5) * P.h;
  for (int c = tid; c < (BX + 1) * BY; c += XTHR) {
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
        int la = fx + y * (BX + 2), lb = la + 1;  // slope slots of cells f-1, f
        double dA = R[F_D * RREG + sa], dB = R[F_D * RREG + sa + 1];
        bool wetA = dA > P.eps, wetB = dB > P.eps;
        if (wetA || wetB) {
          double bA = R[F_B * RREG + sa], bB = R[F_B * RREG + sa + 1];
          double bf = smax(bA, bB);
          SideState L, Rr;
          L.hs = L.hcell = L.un = L.ut = 0.0;
          Rr = L;
          if (wetA) {
            Slopes q = {SL[la], SL[NSL + la], SL[2 * NSL + la]};
            L = side_from_slopes(R[F_E * RREG + sa], R[F_U * RREG + sa], R[F_V * RREG + sa],
                                 R[F_SX * RREG + sa], bA, q, face_p, bf);
          }
          if (wetB) {
            Slopes q = {SL[lb], SL[NSL + lb], SL[2 * NSL + lb]};
            Rr = side_from_slopes(R[F_E * RREG + sa + 1], R[F_U * RREG + sa + 1],
                                  R[F_V * RREG + sa + 1], R[F_SX * RREG + sa + 1], bB, q, face_m,
                                  bf);
          }
          rec = face_from_sides(wetA, wetB, L, Rr, P.g, SP);
          if (!face_finite(rec)) {
            unsigned long long key = fused_flux_key(G, A.bflag, 0, jg, f);
            my_err = key < my_err ? key : my_err;
          }
        }
      }
    }
    FB[0 * NFC + c] = rec.fm;
    FB[1 * NFC + c] = rec.fnl;
    FB[2 * NFC + c] = rec.fnr;
    FB[3 * NFC + c] = rec.ft;
  }
  __syncthreads();
  // face taps (nested-grid flux correction): each tile records its west
  // faces only (fx < BX), so every face is written once; faces no active
  // tile computes stay 0 (dry)
  if (A.taps.n) {
    for (int c = tid; c < (BX + 1) * BY; c += XTHR) {
      const int fx = c % (BX + 1), y = c / (BX + 1), f = i0 + fx, jg = G.jg0 + r0 + y;
      for (int q = 0; q < A.taps.n; ++q)
        if (fx < BX && r0 + y < G.r1 && (f == A.taps.i0[q] || f == A.taps.i0[q] + A.taps.ni[q]) &&
            jg >= A.taps.j0[q] && jg < A.taps.j0[q] + A.taps.nj[q])
          A.taps.out[q][(f == A.taps.i0[q] ? 0 : A.taps.nj[q]) + (jg - A.taps.j0[q])] =
              tau * FB[0 * NFC + c];
    }
  }
  double px_m[PER], px_a[PER], px_c[PER];  // (W.fm-E.fm), (W.fnr-E.fnl), (W.ft-E.ft)
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    int c = tid + m * XTHR;
    if (BX * BY % XTHR && c >= BX * BY) break;
    int x = c % BX, y = c / BX;
    int w = x + y * (BX + 1), e = w + 1;
    px_m[m] = FB[0 * NFC + w] - FB[0 * NFC + e];
    px_a[m] = FB[2 * NFC + w] - FB[1 * NFC + e];
    px_c[m] = FB[3 * NFC + w] - FB[3 * NFC + e];
  }

  // ---- phase 3y: y slopes of rows -1..BY (columns of the tile) -------------
  for (int c = tid; c < BX * (BY + 2); c += XTHR) {
    int x = c % BX, yy = c / BX;
    int r = r0 - 1 + yy, jg = G.jg0 + r;
    int s = (x + 2) + (yy + 1) * RX;
    double se = 0.0, su = 0.0, st = 0.0;
    if (jg > 0 && jg + 1 < G.ny && i0 + x < G.nx && R[F_D * RREG + s] > P.eps) {
      Slopes q = cell_slopes(R[F_E * RREG + s - RX], R[F_V * RREG + s - RX],
                             R[F_U * RREG + s - RX], R[F_SY * RREG + s - RX], R[F_E * RREG + s],
                             R[F_V * RREG + s], R[F_U * RREG + s], R[F_SY * RREG + s],
                             R[F_E * RREG + s + RX], R[F_V * RREG + s + RX],
                             R[F_U * RREG + s + RX], R[F_SY * RREG + s + RX], P.h, SP);
      se = q.eta;
      su = q.un;
      st = q.ut;
    }
    SL[0 * NSL + c] = se;
    SL[1 * NSL + c] = su;
    SL[2 * NSL + c] = st;
  }
  __syncthreads();

  // ---- phase 4y: y faces (stepper.cpp:449-494, 518-538) ----------------------
  for (int c = tid; c < BX * (BY + 1); c += XTHR) {
    int x = c % BX, fy = c / BX;
    int i = i0 + x, rf = r0 + fy;  // face between local rows rf-1 and rf
    int jf = G.jg0 + rf;           // global face index
    FaceRec rec;
    rec.fm = rec.fnl = rec.fnr = rec.ft = 0.0;
    if (i < G.nx && rf <= G.r1) {
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
        int la = x + fy * BX, lb = la + BX;  // slope slots of rows rf-1, rf
        double dA = R[F_D * RREG + sa], dB = R[F_D * RREG + sa + RX];
        bool wetA = dA > P.eps, wetB = dB > P.eps;
        if (wetA || wetB) {
          double bA = R[F_B * RREG + sa], bB = R[F_B * RREG + sa + RX];
          double bf = smax(bA, bB);
          SideState L, Rr;
          L.hs = L.hcell = L.un = L.ut = 0.0;
          Rr = L;
          if (wetA) {
            Slopes q = {SL[la], SL[NSL + la], SL[2 * NSL + la]};
            L = side_from_slopes(R[F_E * RREG + sa], R[F_V * RREG + sa], R[F_U * RREG + sa],
                                 R[F_SY * RREG + sa], bA, q, face_p, bf);
          }
          if (wetB) {
            Slopes q = {SL[lb], SL[NSL + lb], SL[2 * NSL + lb]};
            Rr = side_from_slopes(R[F_E * RREG + sa + RX], R[F_V * RREG + sa + RX],
                                  R[F_U * RREG + sa + RX], R[F_SY * RREG + sa + RX], bB, q,
                                  face_m, bf);
          }
          rec = face_from_sides(wetA, wetB, L, Rr, P.g, SP);
          if (!face_finite(rec)) {
            unsigned long long key = fused_flux_key(G, A.bflag, 1, i, jf);
            my_err = key < my_err ? key : my_err;
          }
        }
      }
    }
    FB[0 * NFC + c] = rec.fm;
    FB[1 * NFC + c] = rec.fnl;
    FB[2 * NFC + c] = rec.fnr;
    FB[3 * NFC + c] = rec.ft;
  }
  __syncthreads();
  if (A.taps.n) {
    for (int c = tid; c < BX * (BY + 1); c += XTHR) {
      const int x = c % BX, fy = c / BX, i = i0 + x, rf = r0 + fy, jf = G.jg0 + rf;
      for (int q = 0; q < A.taps.n; ++q)
        if (fy < BY && i < G.nx && rf < G.r1 &&
            (jf == A.taps.j0[q] || jf == A.taps.j0[q] + A.taps.nj[q]) && i >= A.taps.i0[q] &&
            i < A.taps.i0[q] + A.taps.ni[q])
          A.taps.out[q][2 * A.taps.nj[q] + (jf == A.taps.j0[q] ? 0 : A.taps.ni[q]) +
                        (i - A.taps.i0[q])] = tau * FB[0 * NFC + c];
    }
  }

  // ---- phase 5: accumulate (stepper.cpp:540-566) + final (628-659) ---------
  double deficit = 0.0;
  const double dt_h = tau / P.h;
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    int c = tid + m * XTHR;
    if (BX * BY % XTHR && c >= BX * BY) break;
    int x = c % BX, y = c / BX;
    int i = i0 + x, r = r0 + y;
    if (i >= G.nx || r >= G.r1) continue;
    int jg = G.jg0 + r;
    int s = (x + 2) + (y + 2) * RX;
    size_t k = (size_t)i + (size_t)r * nx;
    const int bc = s_bcol[x], br = s_brow[y];  // i / bs, jg / bs
    unsigned char bfl = bf_staged ? s_bf[(bc - bi_lo) + (br - bj_lo) * nbi]
                                  : A.bflag[bc + (br - G.bj0) * G.nbx];
    bool flux_on = !G.skip || (bfl & 2);
    // the base state k_lag left: the Lagrangian state of an active cell, the
    // step-start state otherwise (stepper.cpp:641-651)
    const double Htm = A.Ho[k], Qxm = A.HUxo[k], Qym = A.HUyo[k];
    if (!flux_on) {  // block skipped by the reference: state unchanged
      peer_store(G, A, i, r, Htm, Qxm, Qym);
      continue;
    }
    int sf = x + y * BX, nf_ = sf + BX;  // S and N face of the cell
    double py_m = FB[0 * NFC + sf] - FB[0 * NFC + nf_];
    double py_a = FB[2 * NFC + sf] - FB[1 * NFC + nf_];  // S.fnr - N.fnl
    double py_c = FB[3 * NFC + sf] - FB[3 * NFC + nf_];  // S.ft - N.ft
    double d = R[F_D * RREG + s];
    bool wet = d > P.eps;
    double cx = 0.0, cy = 0.0;
    if (wet) {
      auto nb = [&](bool in, int q) {
        return SNbr{in, R + F_D * RREG, R + F_E * RREG, R + F_U * RREG, R + F_V * RREG, q};
      };
      double eta_c = R[F_E * RREG + s];
      double gx = eta_grad_comp(nb(i > 0, s - 1), nb(i + 1 < G.nx, s + 1), eta_c, P, SP);
      double gy = eta_grad_comp(nb(jg > 0, s - RX), nb(jg + 1 < G.ny, s + RX), eta_c, P, SP);
      double gh = (P.g * d) * P.h;
      cx = gh * gx;
      cy = gh * gy;
    }
    double Fh = px_m[m] + py_m;
    double Fvx = (px_a[m] + py_c) + cx;
    double Fvy = (py_a + px_c[m]) + cy;
    double H1, qx, qy, dfc;
    final_cell(Htm, Qxm, Qym, Fh, Fvx, Fvy, dt_h, P.eps, H1, qx, qy, dfc);
    deficit += dfc;
    // staged: the base state lives in the output buffers, so a tile whose
    // speculation failed must leave them intact for its exact redo
    SL[c] = H1;
    SL[BX * BY + c] = qx;
    SL[2 * BX * BY + c] = qy;
  }
  const bool any_bad = __syncthreads_or(!sok);
  if (!(SPEC && any_bad)) {
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      int c = tid + m * XTHR;
      if (BX * BY % XTHR && c >= BX * BY) break;
      int x = c % BX, y = c / BX;
      int i = i0 + x, r = r0 + y;
      if (i >= G.nx || r >= G.r1) continue;
      const int bc = s_bcol[x], br = s_brow[y];
      unsigned char bfl = bf_staged ? s_bf[(bc - bi_lo) + (br - bj_lo) * nbi]
                                    : A.bflag[bc + (br - G.bj0) * G.nbx];
      if (G.skip && !(bfl & 2)) continue;
      size_t k = (size_t)i + (size_t)r * nx;
      const double H1 = SL[c], qx = SL[BX * BY + c], qy = SL[2 * BX * BY + c];
      A.Ho[k] = H1;
      A.HUxo[k] = qx;
      A.HUyo[k] = qy;
      if (A.hH) {  // host-buffer step: write the updated cell straight into the caller's arrays
        A.hH[k] = H1;
        A.hHUx[k] = qx;
        A.hHUy[k] = qy;
      }
      peer_store(G, A, i, r, H1, qx, qy);
    }
    if (tid == 0) A.tile_same[tile] = 0;
    // the neighbour reads these rows after a stream-ordered token from us:
    // make the peer stores visible system-wide before this kernel completes
    if (A.peer[0][0] || A.peer[1][0]) __threadfence_system();
  }


  // ---- per-tile diagnostic partials (deterministic) ------------------------
  double v2[2] = {deficit, outflow};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    double v = v2[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) s_red[q][tid >> 5] = v;
  }
  __syncthreads();
  if (tid < 2) {
    double v = 0.0;
    for (int w = 0; w < XTHR / 32; ++w) v += s_red[tid][w];
    A.part[5 * (size_t)tile + 2 * tid] = v;  // [0] deficit, [2] outflow
  }
  if (SPEC && any_bad) {
    if (tid == 0) A.redo[atomicAdd(&sc->redo_n[1], 1)] = tile;
  } else if (my_err != ERR_NONE) {
    atomicMin(&sc->err_key, my_err);
  }
}

__global__ void __launch_bounds__(XTHR, SWF_FLUX_MINB) k_flux_list(Geo G, StepArgs A) {
  __shared__ int s_next;
  StepScalars* sc = A.sc;
  const int n = *(volatile int*)&sc->list_n[1];
  while (true) {
    if (threadIdx.x == 0) s_next = atomicAdd(&sc->list_take[1], 1);
    __syncthreads();
    const int q = s_next;
    __syncthreads();
    if (q >= n) break;
    flux_tile<SWF_SPECULATE != 0>(G, A, A.list[q]);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(XTHR, SWF_FLUX_MINB) k_flux_redo(Geo G, StepArgs A) {
  const int n = *(volatile int*)&A.sc->redo_n[1];
  for (int q = blockIdx.x; q < n; q += gridDim.x) {
    flux_tile<false>(G, A, A.redo[q]);
    __syncthreads();
  }
}

#endif  // !SWF_STEP_SLIM

// ---------------------------------------------------------------------------
// Exact StepInfo volumes (final_update, stepper.cpp:676-701): the reference
// sums the clamp deficit and the source volume per block in row-major cell
// order, then over the flux / Lagrangian blocks in block order, and the
// outflow over the edge faces in a fixed order -- serial floating-point
// sums.  k_step stores the terms that can be nonzero (every cell's deficit
// in the rare tiles with a clamp, Ht - Hn of the active cells of tiles near a
// source spec, the mass flux of each edge face it computes); the tile
// partials, the source masks and the block flags of the step say which
// blocks and cells the reference sums.  These two kernels redo the reference's sums in its order
// on request (a synchronised step or the last step of a run).
// ---------------------------------------------------------------------------
constexpr int XCHUNK = 1024;  // blocks per k_xblock CTA (one nonzero count each)

// Per-block partials of the step's deficit and source-volume terms, in the
// reference's row-major cell order; blocks that cannot hold a nonzero term
// are skipped (no clamp deficit in any tile they touch -- the tile partials
// are sums of non-negative terms -- and no source spec near them).
__global__ void __launch_bounds__(XCHUNK) k_xblock(Geo G, StepArgs A, const double* Hn,
                                                   double* bpart, int* chunk_nz) {
  const StepScalars* sc = A.sc;
  if (stopped(sc)) return;
  const PhysConst& P = G.P;
  const int nbl = G.nbx * (G.bj1 - G.bj0);
  const int lb = blockIdx.x * XCHUNK + threadIdx.x;
  double part[2] = {0.0, 0.0};
  if (lb < nbl) {
    const int bi = lb % G.nbx, bj = G.bj0 + lb / G.nbx;
    const int i0 = bi * G.bs, i1 = min(i0 + G.bs, G.nx);
    const int j0 = bj * G.bs, j1 = min(j0 + G.bs, G.ny);
    const unsigned char f = A.bflag[lb];
    // the fused tiles the block touches (owned rows of this context)
    const int tx0 = i0 / BX, tx1 = (i1 - 1) / BX;
    const int ty0 = (j0 - G.jg0 - G.r0) / BY, ty1 = (j1 - 1 - G.jg0 - G.r0) / BY;
    bool maydef = false, maysrc = false;
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) {
        const int t = tx + ty * G.tiles_x;
        maydef |= A.part[5 * (size_t)t] != 0.0;
        maysrc |= A.tile_srcm[t] != 0u;
      }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      // deficit over the flux blocks, source volume over the Lagrangian ones
      // (stepper.cpp:678-683); every term of such a block was stored this step
      const double* val = q == 0 ? A.xdef : A.xsrc;
      const bool blk = q == 0 ? (!G.skip || (f & 2)) : (!G.skip || (f & 1));
      if (!val || !blk || !(q == 0 ? maydef : maysrc)) continue;
      double acc = 0.0;
      for (int j = j0; j < j1; ++j) {  // row-major, stepper.cpp:633-634 / 345-346
        const size_t row = (size_t)(j - G.jg0) * G.nx;
        const int trow = (j - G.jg0 - G.r0) / BY * G.tiles_x;
        for (int i = i0; i < i1; ++i) {
          // only the tiles that stored their terms this step hold any: a
          // nonzero deficit partial, or a source spec nearby
          const int t = trow + i / BX;
          if (q == 0 ? A.part[5 * (size_t)t] == 0.0 : A.tile_srcm[t] == 0u) continue;
          // the source sum runs over the active cells (cell_active,
          // stepper.hpp:131-133): H_n > eps or a source marker at t_n
          if (q == 1 && !(Hn[row + i] > P.eps ||
                          cell_sigma_only(A.src, A.sig, G.nsrc, i, j) != 0.0))
            continue;
          acc += val[row + i];
        }
      }
      part[q] = acc;
    }
    bpart[2 * (size_t)lb] = part[0];
    bpart[2 * (size_t)lb + 1] = part[1];
  }
  const int nz = __syncthreads_count(part[0] != 0.0 || part[1] != 0.0);
  if (threadIdx.x == 0) chunk_nz[blockIdx.x] = nz;
}

// CTA-wide ordered compaction: thread t contributes terms a (and b) in the
// order (t, a), (t, b); the nonzero ones land in out[] in that order.
// Returns the count (all threads).
__device__ __forceinline__ int cta_compact2(double a, double b, double* out, int* s_warp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = (a != 0.0) + (b != 0.0);
  int incl = c;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {  // scan of the warp totals
    int v = lane < XCHUNK / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < XCHUNK / 32) s_warp[32 + lane] = v;  // inclusive totals
  }
  __syncthreads();
  int pos = (warp > 0 ? s_warp[32 + warp - 1] : 0) + incl - c;
  if (a != 0.0) out[pos++] = a;
  if (b != 0.0) out[pos] = b;
  const int total = s_warp[32 + XCHUNK / 32 - 1];
  __syncthreads();
  return total;
}

// Thread 0's serial sum of n terms in order, loads batched ahead of the
// dependent additions.
__device__ __forceinline__ double serial_add(double acc, const double* v, int n) {
  int q = 0;
  for (; q + 8 <= n; q += 8) {
    double t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = v[q + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += t[u];
  }
  for (; q < n; ++q) acc += v[q];
  return acc;
}

// One CTA: the block-order sums over the nonzero partials and the edge faces
// in the reference's order (stepper.cpp:684-700), then the StepInfo volumes.
// Loads, zero tests and the ordered compaction are parallel; thread 0 adds
// the nonzero terms in order.
__global__ void __launch_bounds__(XCHUNK) k_xserial(Geo G, StepArgs A, const double* bpart,
                                                    const int* chunk_nz, double area, double h) {
  StepScalars* sc = A.sc;
  if (stopped(sc)) return;
  __shared__ double s_c[2][XCHUNK];   // compacted terms (deficit | source, or the faces)
  __shared__ double s_f[2 * XCHUNK];
  __shared__ int s_warp[64];
  __shared__ int s_list[XCHUNK];
  __shared__ int s_n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nbl = G.nbx * (G.bj1 - G.bj0);
  const int nch = (nbl + XCHUNK - 1) / XCHUNK;
  double sum0 = 0.0, sum1 = 0.0, out = 0.0;  // thread 0's running sums
  for (int cb = 0; cb < nch; cb += XCHUNK) {
    // the nonzero chunks of this range, in order
    if (tid == 0) s_n = 0;
    __syncthreads();
    const bool nz = cb + tid < nch && chunk_nz[cb + tid] != 0;
    const unsigned bm = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) s_warp[warp] = (int)bm;
    __syncthreads();
    if (tid == 0) {
      int n = 0;
      for (int w = 0; w < XCHUNK / 32; ++w)
        for (unsigned m = (unsigned)s_warp[w]; m; m &= m - 1) s_list[n++] = cb + 32 * w + __ffs(m) - 1;
      s_n = n;
    }
    __syncthreads();
    const int nlist = s_n;
    for (int li = 0; li < nlist; ++li) {
      const int lb = s_list[li] * XCHUNK + tid;
      const double v0 = lb < nbl ? bpart[2 * (size_t)lb] : 0.0;
      const double v1 = lb < nbl ? bpart[2 * (size_t)lb + 1] : 0.0;
      const int n0 = cta_compact2(v0, 0.0, s_c[0], s_warp);
      const int n1 = cta_compact2(v1, 0.0, s_c[1], s_warp);
      if (tid == 0) {
        sum0 = serial_add(sum0, s_c[0], n0);
        sum1 = serial_add(sum1, s_c[1], n1);
      }
      __syncthreads();
    }
  }
  // out -= W[j]; out += E[j] for every row, then out -= S[i]; out += N[i]
  // (live faces only: the edge cell's block is flux-active, stepper.cpp:684-688)
  auto live = [&](int ci, int cj) {
    return !G.skip || (A.bflag[ci / G.bs + (cj / G.bs - G.bj0) * G.nbx] & 2);
  };
  for (int pass = 0; pass < 2; ++pass) {
    const int n = pass == 0 ? G.ny : G.nx;
    const int lo = pass == 0 ? 0 : 2 * G.ny, hi = pass == 0 ? G.ny : 2 * G.ny + G.nx;
    for (int base = 0; base < n; base += XCHUNK) {
      const int q = base + tid;
      double w = 0.0, e = 0.0;
      if (q < n) {
        if (pass == 0 ? live(0, q) : live(q, 0)) w = A.xface[lo + q];
        if (pass == 0 ? live(G.nx - 1, q) : live(q, G.ny - 1)) e = A.xface[hi + q];
      }
      const int nf = cta_compact2(-w, e, s_f, s_warp);  // out -= w is out + (-w), exactly
      if (tid == 0) out = serial_add(out, s_f, nf);
      __syncthreads();
    }
  }
  if (tid == 0) {
    sc->deficit = sum0 * area;           // stepper.cpp:680
    sc->srcvol = sum1 * area;            // stepper.cpp:683
    sc->outflow = (out * sc->tau) * h;   // stepper.cpp:701
  }
}

// k_reduce: RED_CTAS fixed-order partial sums of the per-tile partials
// (deficit, source volume, outflow, Lagrangian blocks, flux blocks; coalesced,
// deterministic); k_finish adds them in CTA order and commits t.
constexpr int NPART = 5;
__global__ void k_reduce(const double* part, int ntiles, double* red, const StepScalars* sc) {
  __shared__ double s[NPART][NTHR];
  double v[NPART] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (!stopped(sc)) {
    int chunk = (ntiles + gridDim.x - 1) / gridDim.x;
    int a = blockIdx.x * chunk, e = min(a + chunk, ntiles);
    for (int t = a + threadIdx.x; t < e; t += NTHR)
#pragma unroll
      for (int q = 0; q < NPART; ++q) v[q] += part[NPART * (size_t)t + q];
  }
  for (int q = 0; q < NPART; ++q) s[q][threadIdx.x] = v[q];
  __syncthreads();
  for (int w = NTHR / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int q = 0; q < NPART; ++q) s[q][threadIdx.x] += s[q][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < NPART) red[NPART * blockIdx.x + threadIdx.x] = s[threadIdx.x][0];
}

// One CTA: the partials are staged in shared memory by all threads (one
// round of loads instead of nred dependent ones), then thread 0 sums them in
// the same fixed order as ever.
__global__ void k_finish(const double* red, int nred, StepScalars* sc, double area, double h,
                         int counts_from_tiles) {
  __shared__ double s_red[NPART * RED_CTAS];
  if (stopped(sc)) {
    if (threadIdx.x == 0 && sc->fail_step < 0) sc->fail_step = sc->steps_done;
    return;
  }
  for (int i = threadIdx.x; i < NPART * nred; i += blockDim.x) s_red[i] = red[i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double w[NPART] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int t = 0; t < nred; ++t)
    for (int q = 0; q < NPART; ++q) w[q] += s_red[NPART * t + q];
  sc->deficit = w[0] * area;
  sc->srcvol = w[1] * area;
  sc->outflow = (w[2] * sc->tau) * h;
  if (counts_from_tiles) {
    sc->lag_act = (int)w[3];
    sc->flux_act = (int)w[4];
  }
  sc->t_prev = sc->t;
  sc->t += sc->tau;  // stepper.cpp:703
  sc->steps_done += 1;
  sc->mask_valid = 1;
}

StepArgs step_args(swf_ctx* c) {
  StepArgs A;
  A.taps = c->taps;
  for (int side = 0; side < 2; ++side) {
    for (int f = 0; f < 3; ++f) A.peer[side][f] = c->peer_on[side] ? c->peer[side][f][1 - c->cur] : nullptr;
    A.peer_drow[side] = c->peer_drow[side];
  }
  A.hH = c->wt_host[0];
  A.hHUx = c->wt_host[1];
  A.hHUy = c->wt_host[2];
  int cur = c->cur, nxt = 1 - c->cur;
  A.H = c->H[cur];
  A.HUx = c->HUx[cur];
  A.HUy = c->HUy[cur];
  A.b = c->b;
  A.nf = c->nf;
  A.fpx = c->fpx;
  A.fpy = c->fpy;
  A.lamn = c->d_lamn;
  A.gxy = c->d_gxy;
  A.Ho = c->H[nxt];
  A.HUxo = c->HUx[nxt];
  A.HUyo = c->HUy[nxt];
  A.src = c->d_src;
  A.sig = c->d_sig;
  A.bflag = c->d_bflag;
  A.tile_act = tile_act_at(c, c->cur);
  A.tile_same = c->d_tile_same;
  A.tile_srcm = c->d_tile_srcm;
  A.redo = c->d_redo_s;
  A.list = c->d_list_s;
  A.part = c->d_part;
  A.sc = c->d_sc;
  A.hd = c->d_half[0];
  A.hu = c->d_half[1];
  A.hv = c->d_half[2];
  A.redo_l = c->d_redo_l;
  A.xdef = c->d_xdef;
  A.xsrc = c->geo.nsrc > 0 ? c->d_xsrc : nullptr;
  A.xface = c->d_xface;
  return A;
}

// The TMA descriptors of this step: the step-start buffer (cur) and b.
TmaArgs tma_args(const swf_ctx* c) {
  TmaArgs T;
  T.on = (SWF_TMA && SWF_STEP_SLIM && c->tma_ok) ? 1 : 0;
  for (int q = 0; q < 3; ++q) T.m[q] = c->tma_state[c->cur][q];
  T.m[3] = c->tma_b;
  return T;
}

constexpr size_t step_smem() {
  return (size_t)(F_NUM * RREG + SCRATCH) * sizeof(double);
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

bool mask_fused(const Geo& G) { return G.bs <= 16 && 16 % G.bs == 0; }

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
  if (nt > 0)
    k_tiles<<<(nt + 127) / 128, 128, 0, c->stream>>>(G, c->d_bflag, tile_act_at(c, c->cur),
                                                     c->d_sc);
  return cuda_check(c, cudaGetLastError(), "k_mask");
}

int launch_tau(swf_ctx* c, double dt_cap) {
  k_tau<<<1, 1, 0, c->stream>>>(c->geo, c->d_src, c->d_ht, c->d_hq, c->d_wt, c->d_wv, c->d_sig,
                                c->d_sc, dt_cap, -1.0, nullptr);
  return cuda_check(c, cudaGetLastError(), "k_tau");
}

int launch_mid(swf_ctx* c, double tau) {
  k_mid<<<1, 1, 0, c->stream>>>(c->geo, c->d_src, c->d_ht, c->d_hq, c->d_wt, c->d_wv, c->d_sig,
                                c->d_sc, tau);
  return cuda_check(c, cudaGetLastError(), "k_mid");
}

// part: -1 = the whole phase (begin + every forces tile row); -2 = every
// forces tile row, k_begin (and k_mask) already enqueued by the caller (the
// host-buffer strip step); 0 = begin + the tile rows that read no ghost row
// (a strip's interior, computable while its halo exchange is in flight);
// 1 = the remaining (ghost-dependent) rows.
int fused_enqueue_phase1(swf_ctx* c, double dt_cap, int part) {
  NvtxRange nv("swf:forces (K1-K3)");
  const Geo& G = c->geo;
  int rc;
  bool fm = mask_fused(G);
  // The interior/ghost split needs the block mask inside k_forces (block
  // sizes dividing 16); otherwise k_mask reads the ghost rows, so the whole
  // phase 1 runs in the second (post-exchange) part and the first is empty --
  // the same results, without the overlap.
  if (!fm && part == 0) return SWF_OK;
  if (!fm && part == 1) part = -1;
  if (part == -2) {
    part = -1;
  } else if (part <= 0) {
    ev(c, 0);
    if ((rc = launch_begin(c, dt_cap))) return rc;
    if (!fm && (rc = launch_mask(c))) return rc;
    ev(c, 1);
  }
  ForcesArgs A;
  A.H = c->H[c->cur];
  A.HUx = c->HUx[c->cur];
  A.HUy = c->HUy[c->cur];
  A.b = c->b;
  A.nf = c->nf;
  A.src = c->d_src;
  A.sig = c->d_sig;
  A.fpx = c->fpx;
  A.fpy = c->fpy;
  A.lamn = c->d_lamn;
  A.interior = c->d_interior;
  A.halo = c->d_halo;
  A.bflag = c->d_bflag;
  A.tile_act = tile_act_at(c, c->cur);
  A.tile_prev = tile_act_at(c, 1 - c->cur);
  A.tile_srcm = c->d_tile_srcm;
  A.redo = c->d_redo_f;
  A.list = c->d_list_f;
  A.sc = c->d_sc;
  A.cnt_part = c->d_part;
  forces_rows(c, A.ra0, A.ra1);
  A.tr_lo = -((G.r0 - A.ra0 + BY - 1) / BY);
  int tr_hi = (A.ra1 - G.r0 + BY - 1) / BY;
  if (tr_hi < G.tiles_y) tr_hi = G.tiles_y;
  A.do_mask = fm ? 1 : 0;
  A.lr0 = A.tr_lo;
  A.lr1 = tr_hi;
  // the work list + persistent grid (k_flist / k_forces_list) over tile rows
  // [r_first, r_end); one CTA per tile when the mask is not fused
  auto listed = [&](int r_first, int r_end) {
    if (r_end <= r_first) return;
    ForcesArgs B = A;
    B.lr0 = r_first;
    B.lr1 = r_end;
    int ntile = G.tiles_x * (r_end - r_first);
    if (SWF_TILE_LISTS && fm) {
      k_flist<<<(ntile + 255) / 256, 256, 0, c->stream>>>(G, B);
      k_forces_list<<<c->sm_count * SWF_FORCES_MINB, FTHR, 0, c->stream>>>(G, B);
    } else {
      B.tr_lo = r_first;
      k_forces<<<ntile, FTHR, 0, c->stream>>>(G, B);
    }
  };
  if (part < 0) {
    int ntile = G.tiles_x * (tr_hi - A.tr_lo);
    listed(A.tr_lo, tr_hi);
    if (ntile > 0 && SWF_SPECULATE) k_forces_redo<<<RED_CTAS, FTHR, 0, c->stream>>>(G, A);
  } else {
    // interior tile rows [a, b): their 1-row halo stays inside the owned rows
    int a = G.r0 > 0 ? 1 : 0;
    int b = G.r1 < G.rows ? G.tiles_y - 1 : G.tiles_y;
    if (b < a) b = a;
    const int lo = A.tr_lo;
    auto launch = [&](int r_first, int r_end) {
      if (r_end <= r_first) return;
      ForcesArgs B = A;
      B.tr_lo = r_first;
      k_forces<<<G.tiles_x * (r_end - r_first), FTHR, 0, c->stream>>>(G, B);
    };
    if (part == 0) {
      listed(a, b);  // interior rows: the list (one list per step, k_begin reset it)
    } else {
      launch(lo, a);
      launch(b, tr_hi);
      if (SWF_SPECULATE) k_forces_redo<<<RED_CTAS, FTHR, 0, c->stream>>>(G, A);
    }
  }
  if (part != 0) ev(c, 2);
  return cuda_check(c, cudaGetLastError(), "k_forces");
}

int fused_enqueue_phase1(swf_ctx* c, double dt_cap) { return fused_enqueue_phase1(c, dt_cap, -1); }

// this context's CFL speed (max over the per-CTA slots) into a device double
__global__ void k_local_speed(const StepScalars* sc, double* out) {
  if (stopped(sc)) {  // the stop travels through the speed allreduce
    *out = bitsd(SPEED_STOP_BITS);
    return;
  }
  unsigned long long mb = sc->speed_bits;
  for (int q = 0; q < SPEED_SLOTS; ++q) mb = sc->speed_slots[q] > mb ? sc->speed_slots[q] : mb;
  *out = bitsd(mb);
}

int fused_local_speed(swf_ctx* c, double* dev_out) {
  k_local_speed<<<1, 1, 0, c->stream>>>(c->d_sc, dev_out);
  return cuda_check(c, cudaGetLastError(), "k_local_speed");
}

int fused_enqueue_phase2(swf_ctx* c, double dt_cap, double global_speed, const double* gspeed) {
  NvtxRange nv("swf:step (tau, K4-K8, diagnostics)");
  const Geo& G = c->geo;
  k_tau<<<1, 1, 0, c->stream>>>(G, c->d_src, c->d_ht, c->d_hq, c->d_wt, c->d_wv, c->d_sig,
                                c->d_sc, dt_cap, global_speed, gspeed);
  ev(c, 3);
  int nt = G.tiles_x * G.tiles_y;
  for (int q = 0; q < c->taps.n; ++q)
    cudaMemsetAsync(c->taps.out[q], 0,
                    2 * (size_t)(c->taps.ni[q] + c->taps.nj[q]) * sizeof(double), c->stream);
#if !SWF_STEP_SLIM
  if (nt > 0 && SWF_TILE_LISTS && SWF_SPLIT) {
    StepArgs SA = step_args(c);
    k_slist<<<(nt + 255) / 256, 256, 0, c->stream>>>(G, SA);
    k_lag_list<<<c->sm_count * SWF_LAG_MINB, LTHR, lag_smem(), c->stream>>>(G, SA);
    if (SWF_SPECULATE) k_lag_redo<<<RED_CTAS, LTHR, lag_smem(), c->stream>>>(G, SA);
    if (G.r0 > 0 || G.r1 < G.rows)
      k_ghost_half<<<(4 * G.nx + 127) / 128, 128, 0, c->stream>>>(G, SA);
    k_flux_list<<<c->sm_count * SWF_FLUX_MINB, XTHR, flux_smem(), c->stream>>>(G, SA);
    if (SWF_SPECULATE) k_flux_redo<<<RED_CTAS, XTHR, flux_smem(), c->stream>>>(G, SA);
  } else
#endif
  {
    if (nt > 0 && SWF_TILE_LISTS) {
      StepArgs SA = step_args(c);
      k_slist<<<(nt + 255) / 256, 256, 0, c->stream>>>(G, SA);
      k_step_list<<<c->sm_count * SWF_STEP_MINB, STHR, step_smem(), c->stream>>>(G, SA,
                                                                                 tma_args(c));
    } else if (nt > 0) {
      k_step<<<nt, STHR, step_smem(), c->stream>>>(G, step_args(c), tma_args(c));
    }
    if (nt > 0 && SWF_SPECULATE)
      k_step_redo<<<RED_CTAS, STHR, step_smem(), c->stream>>>(G, step_args(c), tma_args(c));
  }
  ev(c, 4);
  double* red = c->d_part + NPART * (size_t)(nt > 0 ? nt : 1);
  k_reduce<<<RED_CTAS, NTHR, 0, c->stream>>>(c->d_part, nt, red, c->d_sc);
  k_finish<<<1, NTHR, 0, c->stream>>>(red, RED_CTAS, c->d_sc, c->h * c->h, c->h,
                                   mask_fused(G) ? 1 : 0);
  ev(c, 5);
  if (c->timing && c->tslots > 0) ++c->tstep;
  c->cur = 1 - c->cur;  // optimistic; rolled back by the caller on failure
  return cuda_check(c, cudaGetLastError(), "k_step");
}

int fused_enqueue_phase2(swf_ctx* c, double dt_cap) {
  return fused_enqueue_phase2(c, dt_cap, -1.0, nullptr);
}
int fused_enqueue_phase2(swf_ctx* c, double dt_cap, double global_speed) {
  return fused_enqueue_phase2(c, dt_cap, global_speed, nullptr);
}

int fused_enqueue_step(swf_ctx* c, double dt_cap) {
  int rc = fused_enqueue_phase1(c, dt_cap);
  if (rc) return rc;
  return fused_enqueue_phase2(c, dt_cap, -1.0, nullptr);
}

// Zero-copy result write-back for the host-buffer step: the cells of the
// tiles k_step updated are stored straight into pinned host memory over
// PCIe; every other tile kept its step-start state, which the caller's
// arrays already hold.  `flags` are the tile flags of the step just run.
__global__ void k_scatter_host(Geo G, const unsigned char* __restrict__ flags,
                               const double* __restrict__ H, const double* __restrict__ HUx,
                               const double* __restrict__ HUy, double* hH, double* hHUx,
                               double* hHUy) {
  const int nt = G.tiles_x * G.tiles_y;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    if (!(flags[t] & 2)) continue;
    int i0 = (t % G.tiles_x) * BX, r0 = G.r0 + (t / G.tiles_x) * BY;
    for (int c = threadIdx.x; c < BX * BY; c += blockDim.x) {
      int i = i0 + c % BX, r = r0 + c / BX;
      if (i >= G.nx || r >= G.r1) continue;
      size_t k = (size_t)i + (size_t)r * G.nx;
      hH[k] = H[k];
      hHUx[k] = HUx[k];
      hHUy[k] = HUy[k];
    }
  }
}

// After an aborted write-through step: the caller's arrays get the step-start
// state (the buffer the step read) back in every tile the step may have
// written, so a numerical abort leaves them as they were.
int fused_restore_host(swf_ctx* c, double* hH, double* hHUx, double* hHUy) {
  const Geo& G = c->geo;
  int cur = c->cur;  // not flipped: the failed step read this buffer; its flags are at cur
  k_scatter_host<<<148 * 8, NTHR, 0, c->stream>>>(G, tile_act_at(c, cur), c->H[cur], c->HUx[cur],
                                                  c->HUy[cur], hH, hHUx, hHUy);
  return cuda_check(c, cudaGetLastError(), "k_restore_host");
}



// Sparse ingest of the momentum for a host-buffer step (swf_step_host on
// pinned arrays): after the depth was copied in full and the block mask
// computed, only the flux-active tiles' HUx, HUy are read from the caller's
// pinned arrays (zero-copy PCIe reads, 16-byte vectors along rows).  Every
// cell whose momentum the step reads or writes back lies in such a tile: a
// wet or source cell makes its block Lagrangian-active, and the write-back
// covers flux-active tiles only.
__global__ void k_ingest_hu(Geo G, const unsigned char* __restrict__ flags,
                            const double* __restrict__ hHUx, const double* __restrict__ hHUy,
                            double* __restrict__ HUx, double* __restrict__ HUy) {
  const int nt = G.tiles_x * G.tiles_y;
  const bool vec = (G.nx % 2 == 0) && ((((uintptr_t)hHUx) | ((uintptr_t)hHUy)) % 16 == 0);
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    if (!(flags[t] & 2)) continue;
    int i0 = (t % G.tiles_x) * BX, r0 = G.r0 + (t / G.tiles_x) * BY;
    if (vec) {
      for (int c = threadIdx.x; c < BX * BY / 2; c += blockDim.x) {
        int i = i0 + 2 * (c % (BX / 2)), r = r0 + c / (BX / 2);
        if (i >= G.nx || r >= G.r1) continue;  // nx even: i + 1 < nx too
        size_t k = (size_t)i + (size_t)r * G.nx;
        *(double2*)(HUx + k) = *(const double2*)(hHUx + k);
        *(double2*)(HUy + k) = *(const double2*)(hHUy + k);
      }
    } else {
      for (int c = threadIdx.x; c < BX * BY; c += blockDim.x) {
        int i = i0 + c % BX, r = r0 + c / BX;
        if (i >= G.nx || r >= G.r1) continue;
        size_t k = (size_t)i + (size_t)r * G.nx;
        HUx[k] = hHUx[k];
        HUy[k] = hHUy[k];
      }
    }
  }
}

int fused_ingest_hu(swf_ctx* c, const double* hHUx, const double* hHUy) {
  k_ingest_hu<<<148 * 8, NTHR, 0, c->stream>>>(c->geo, tile_act_at(c, c->cur), hHUx, hHUy,
                                               c->HUx[c->cur], c->HUy[c->cur]);
  return cuda_check(c, cudaGetLastError(), "k_ingest_hu");
}

size_t fused_tile_bytes() { return step_smem(); }

#ifdef SWF_PHASE_TIMING
extern "C" int swf_debug_phase_cycles(unsigned long long* out16, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, g_phase_cycles, 16 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
  }
  return (int)cudaGetLastError();
}
#endif
int fused_reduce_ctas() { return RED_CTAS; }

// The exact StepInfo volumes of the last enqueued step (full grids; the
// strips keep the deterministic tile-order sums of k_finish).
int fused_exact_volumes(swf_ctx* c) {
  if (!c->d_xdef || SWF_SPLIT) return SWF_OK;
  const Geo& G = c->geo;
  StepArgs A = step_args(c);
  const int nbl = G.nbx * (G.bj1 - G.bj0);
  // the step just enqueued flipped cur: its step-start depth is the other buffer
  const int nch = (nbl + XCHUNK - 1) / XCHUNK;
  int* chunk_nz = (int*)(c->d_xbpart + 2 * (size_t)nbl);  // after the partials
  if (nbl > 0)
    k_xblock<<<nch, XCHUNK, 0, c->stream>>>(G, A, c->H[1 - c->cur], c->d_xbpart, chunk_nz);
  k_xserial<<<1, XCHUNK, 0, c->stream>>>(G, A, c->d_xbpart, chunk_nz, c->h * c->h, c->h);
  return cuda_check(c, cudaGetLastError(), "exact volumes");
}

// Per-tile source masks (bit s: spec s meets the tile's cells +- 2), the
// host-side equivalent of src_mask_for, refreshed whenever the specs change.
int fused_tile_srcm(swf_ctx* c) {
  const Geo& G = c->geo;
  size_t nt = (size_t)G.tiles_x * G.tiles_y;
  std::vector<unsigned> m(nt ? nt : 1, 0u);
  for (size_t t = 0; t < nt; ++t) {
    int tx = (int)(t % G.tiles_x), ty = (int)(t / G.tiles_x);
    int ci0 = tx * BX - 2, ci1 = tx * BX + BX + 1;
    int cj0 = G.jg0 + G.r0 + ty * BY - 2, cj1 = G.jg0 + G.r0 + ty * BY + BY + 1;
    unsigned v = 0;
    if (G.nsrc > 32) {
      v = 0xffffffffu;
    } else {
      for (int q = 0; q < G.nsrc; ++q) {
        const DevSrc& d = c->h_src[q];
        if (d.i0 <= ci1 && d.i1 >= ci0 && d.j0 <= cj1 && d.j1 >= cj0) v |= 1u << q;
      }
    }
    m[t] = v;
  }
  cudaError_t e = cudaSuccess;
  if (!c->d_tile_srcm) e = cudaMalloc(&c->d_tile_srcm, m.size() * sizeof(unsigned));
  if (e == cudaSuccess)
    e = cudaMemcpy(c->d_tile_srcm, m.data(), m.size() * sizeof(unsigned), cudaMemcpyHostToDevice);
  return cuda_check(c, e, "tile source masks");
}

// Kernel attributes must be set outside stream capture (a CUDA graph does not
// record cudaFuncSetAttribute), so contexts call this at creation.
// The reciprocal refinements of h and 2h (eta_grad_comp's divisors) depend
// on the terrain only: refined once here on the device and carried in Geo,
// instead of by every thread of every tile kernel.
__global__ void k_recips(double h, double two_h, double* out) {
  out[0] = recip_of(h).r;
  out[1] = recip_of(two_h).r;
}

int fused_prepare(swf_ctx* c) {
  double* d = nullptr;
  double r[2] = {0.0, 0.0};
  cudaError_t e = cudaMalloc(&d, 2 * sizeof(double));
  if (e == cudaSuccess) {
    k_recips<<<1, 1, 0, c->stream>>>(c->geo.P.h, c->geo.P.two_h, d);
    e = cudaMemcpyAsync(r, d, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(d);
  }
  if (e == cudaSuccess) {
    // outside the normal range the speculative fast path could mistake
    // +0 / h; r = 0 makes every such quotient fail acceptance instead
    double h = c->geo.P.h;
    bool normal = h >= 0x1p-999 && h <= 0x1p999;
    c->geo.P.rh.r = normal ? r[0] : 0.0;
    c->geo.P.r2h.r = normal ? r[1] : 0.0;
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)step_smem());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_step_redo, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)step_smem());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_step_list, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)step_smem());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_step_list, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_forces_list, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e == cudaSuccess) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    c->sm_count = sms > 0 ? sms : 148;
  }
  // redo lists: every owned tile, plus the ghost tile rows k_forces covers
  size_t nredo = (size_t)c->geo.tiles_x * (c->geo.tiles_y + 2 * REDO_ROW0);
  if (e == cudaSuccess && !c->d_redo_f) e = cudaMalloc(&c->d_redo_f, nredo * sizeof(int));
  if (e == cudaSuccess && !c->d_redo_s) e = cudaMalloc(&c->d_redo_s, nredo * sizeof(int));
  if (e == cudaSuccess && !c->d_list_f) e = cudaMalloc(&c->d_list_f, nredo * sizeof(int));
  if (e == cudaSuccess && !c->d_list_s) e = cudaMalloc(&c->d_list_s, nredo * sizeof(int));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_step, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
#if !SWF_STEP_SLIM
  // split step: its kernels' shared memory and the half-step view planes
  for (auto f : {(const void*)k_lag_list, (const void*)k_lag_redo}) {
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lag_smem());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  for (auto f : {(const void*)k_flux_list, (const void*)k_flux_redo}) {
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)flux_smem());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
#endif
  if (e == cudaSuccess && SWF_SPLIT && !c->d_redo_l) e = cudaMalloc(&c->d_redo_l, nredo * sizeof(int));
  if (e == cudaSuccess && SWF_GRAD_SHARE && !c->d_gxy) {
    const size_t bytes = 2 * (local_cells(c) ? local_cells(c) : 1) * sizeof(double);
    e = cudaMalloc(&c->d_gxy, bytes);
    if (e == cudaSuccess) e = cudaMemset(c->d_gxy, 0, bytes);
  }
  if (e == cudaSuccess && SWF_LAMBDA_SHARE && !c->d_lamn) {
    const size_t bytes = (local_cells(c) ? local_cells(c) : 1) * sizeof(double);
    e = cudaMalloc(&c->d_lamn, bytes);
    if (e == cudaSuccess) e = cudaMemset(c->d_lamn, 0, bytes);
  }
  // TMA descriptors of k_step's region loads (2D tiles RX x RY of doubles):
  // the row stride must be a multiple of 16 bytes (even nx); else the
  // per-thread loads stay
  c->tma_ok = 0;
  if (e == cudaSuccess && SWF_TMA && SWF_STEP_SLIM && c->geo.nx % 2 == 0) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn) {
      auto encode = reinterpret_cast<EncodeFn>(fn);
      const cuuint64_t dims[2] = {(cuuint64_t)c->geo.nx, (cuuint64_t)c->geo.rows};
      const cuuint64_t strides[1] = {(cuuint64_t)c->geo.nx * sizeof(double)};
      const cuuint32_t box[2] = {(cuuint32_t)RX, (cuuint32_t)RY};
      const cuuint32_t estr[2] = {1, 1};
      auto mk = [&](CUtensorMap* m, const double* ptr) {
        return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)ptr, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      (CUtensorMapL2promotion)SWF_TMA_L2PROMO,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      };
      bool ok = mk(&c->tma_b, c->b);
      for (int p = 0; p < 2 && ok; ++p)
        ok = mk(&c->tma_state[p][0], c->H[p]) && mk(&c->tma_state[p][1], c->HUx[p]) &&
             mk(&c->tma_state[p][2], c->HUy[p]);
      c->tma_ok = ok ? 1 : 0;
    }
    cudaGetLastError();
  }
  // exact-diagnostics captures: full grids only (a strip's sums continue
  // its neighbours' running totals, which stay with the tile-order sums)
  const bool full = c->geo.r0 == 0 && c->geo.r1 == c->geo.rows;
  if (e == cudaSuccess && full && !SWF_SPLIT && !c->d_xdef) {
    const size_t n = local_cells(c) ? local_cells(c) : 1;
    const size_t nbl = (size_t)c->geo.nbx * (c->geo.bj1 - c->geo.bj0) + 1;
    const size_t nf = 2 * ((size_t)c->geo.nx + c->geo.ny);
    void** bufs[] = {(void**)&c->d_xdef, (void**)&c->d_xsrc, (void**)&c->d_xbpart,
                     (void**)&c->d_xface};
    const size_t sz[] = {n * 8, n * 8, 2 * nbl * 8 + (nbl / XCHUNK + 2) * 4, nf * 8};
    for (int q = 0; q < 4 && e == cudaSuccess; ++q) {
      e = cudaMalloc(bufs[q], sz[q]);
      if (e == cudaSuccess) e = cudaMemset(*bufs[q], 0, sz[q]);
    }
  }
  for (int q = 0; q < 3 && e == cudaSuccess && SWF_SPLIT; ++q) {
    if (c->d_half[q]) continue;
    const size_t bytes = (local_cells(c) ? local_cells(c) : 1) * sizeof(double);
    e = cudaMalloc(&c->d_half[q], bytes);
    if (e == cudaSuccess) e = cudaMemset(c->d_half[q], 0, bytes);
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_forces, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  return cuda_check(c, e, "kernel attributes");
}

}  // namespace swf
