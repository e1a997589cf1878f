// swf_nest.cu — two-level nested grids (zoom-in windows) on the device.
//
// SPEC.md [MODULE] nesting (paper §2.2, §5): a fine window
// of r x r cells per coarse cell, embedded in the global grid, coupled every
// global step: prolong_boundary (coarse -> fine ghost band), subcycling of
// the fine grid with dt_cap so it lands exactly on the coarse time,
// restrict_feedback (fine -> coarse window).  The reference ships NO code for
// this module, so the operator details below are this
// repository's, stated once here and restated by the test oracle
// (oracle/nest.py), which the GPU path matches bit for bit:
//
//  * fine grid = the window at h/r plus a ghost band of `ghost` fine cells on
//    every side: nxf = r*ni + 2*ghost, nyf = r*nj + 2*ghost.  Fine cell
//    (fi, fj) has its centre at coarse index coordinates
//        xc = (i0 + ((fi - ghost) + 0.5) / r) - 0.5   (yc likewise)
//  * prolongation: bilinear in eta = H + b and in HUx, HUy
//    over the 4 surrounding coarse cells, lerp(a, b, t) = a + t*(b - a)
//    (exact on constants: lake at rest stays at rest), x first then y, when
//    all 4 are wet (H > eps); with 1-3 wet cells, the bilinear weights
//    (1-tx)(1-ty), tx(1-ty), (1-tx)ty, tx ty renormalised over the wet cells
//    (a dry cell's eta = b is not a water level: mixing it in would flood a
//    dry fine bed below the coarse one); no wet cell -> dry.
//    H = max(0, eta - b_fine); HU = 0 where H <= eps_dry.  A fine centre on
//    a coarse centre (tx = ty = 0, odd r) takes that cell's depth form
//    H = H_c + (b_c - b_fine), the same value without the (H + b) - b
//    rounding, so r = 1 copies the window exactly.
//  * subcycling: ghosts at fine time tf are
//    lerp(G(t0), G(t1), (tf - t0)/(t1 - t0)) of the two prolongations around
//    the global step; the fine grid steps with dt_cap = tau_g (first
//    substep) or t1 - tf until it is within max(1e-9 tau_g, 8 ulp(t1)) of
//    t1, then its t is set to t1.
//  * restriction: each window cell's H, HUx, HUy = the sum
//    of its r x r fine cells (row-major, j outer) divided by r*r.
//  * flux correction (two-way; the SPEC's mass invariant): the
//    k_step face taps record tau*fm through the window boundary faces of the
//    coarse step and of every fine substep; after the restriction each
//    coarse cell just outside the window trades the coarse face volume for
//    the fine one (k_reflux), so the coupled system is conservative.
//
// After any external write the fused path's dry-tile bookkeeping is updated
// for the touched tiles only (tile flags of the previous step set active, the
// "both ping-pong buffers equal" flag cleared), so dry-block skipping stays
// exact without a full-grid recount.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "swf_internal.cuh"

struct swf_nest {
  swf_ctx* coarse = nullptr;
  swf_ctx* fine = nullptr;
  swf_nest_desc d{};
  int nxf = 0, nyf = 0;
  size_t nghost = 0;  // ghost cells of the fine grid
  double* g[2] = {nullptr, nullptr};  // prolonged ghosts at t0 / t1: [H | HUx | HUy]
  // flux correction (two-way): tau*fm through the window boundary faces of
  // the coarse step and of every fine substep (face taps of k_step)
  double* tap_c = nullptr;      // coarse faces: 2*(ni+nj)
  double* tap_f = nullptr;      // fine faces of one substep: 2*r*(ni+nj)
  double* tap_fsum = nullptr;   // their sum over the substeps
  double* clampv = nullptr;     // per boundary face: volume added by the reflux clamp
  double* d_sub = nullptr;      // device subcycling scalars: [alpha, smallest fine tau]
  int last_subs = 0;            // substeps of the previous coupled step (batch size hint)
  std::string err;
};

namespace swf {
namespace {

constexpr int TBX = 32, TBY = 16;  // fused tile (swf_fused.cu BX, BY)

struct NestGeo {
  int cnx, cny;        // coarse grid
  int i0, j0, ni, nj;  // window (coarse cells)
  int r, gw;           // refinement, ghost band width (fine cells)
  int nxf, nyf;        // fine grid
  double eps;          // eps_dry of the fine grid
  long long nghost;
};

__device__ __forceinline__ double lerp(double a, double b, double t) { return a + t * (b - a); }

// ghost cell q -> fine (fi, fj): gw bottom rows, gw top rows, then the left
// and right gw columns of the middle rows
__device__ __forceinline__ void ghost_cell(const NestGeo& N, long long q, int& fi, int& fj) {
  long long band = (long long)N.gw * N.nxf;
  if (q < band) {
    fj = (int)(q / N.nxf);
    fi = (int)(q % N.nxf);
    return;
  }
  q -= band;
  if (q < band) {
    fj = N.nyf - N.gw + (int)(q / N.nxf);
    fi = (int)(q % N.nxf);
    return;
  }
  q -= band;
  int w2 = 2 * N.gw;
  fj = N.gw + (int)(q / w2);
  int c = (int)(q % w2);
  fi = c < N.gw ? c : N.nxf - w2 + c;
}

__device__ __forceinline__ double coarse_coord(int w0, int f, int gw, int r) {
  return ((double)w0 + ((double)(f - gw) + 0.5) / (double)r) - 0.5;
}

// prolong_boundary: coarse state -> ghost values (one thread per ghost cell)
__global__ void k_prolong(NestGeo N, const double* __restrict__ cH, const double* __restrict__ cU,
                          const double* __restrict__ cV, const double* __restrict__ cb,
                          const double* __restrict__ fb, double* __restrict__ out) {
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= N.nghost) return;
  int fi, fj;
  ghost_cell(N, q, fi, fj);
  double xc = coarse_coord(N.i0, fi, N.gw, N.r), yc = coarse_coord(N.j0, fj, N.gw, N.r);
  int ia = (int)floor(xc), ja = (int)floor(yc);
  double tx = xc - (double)ia, ty = yc - (double)ja;
  size_t k[4];
  k[0] = (size_t)ia + (size_t)ja * N.cnx;
  k[1] = k[0] + 1;
  k[2] = k[0] + N.cnx;
  k[3] = k[2] + 1;
  double h[4], e[4], uu[4], vv[4];
  int nwet = 0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    h[m] = cH[k[m]];
    e[m] = h[m] + cb[k[m]];
    uu[m] = cU[k[m]];
    vv[m] = cV[k[m]];
    nwet += h[m] > N.eps;
  }
  double eta = 0.0, u = 0.0, v = 0.0;
  bool has = true;
  if (nwet == 4) {
    eta = lerp(lerp(e[0], e[1], tx), lerp(e[2], e[3], tx), ty);
    u = lerp(lerp(uu[0], uu[1], tx), lerp(uu[2], uu[3], tx), ty);
    v = lerp(lerp(vv[0], vv[1], tx), lerp(vv[2], vv[3], tx), ty);
  } else if (nwet == 0) {
    has = false;
  } else {  // bilinear weights renormalised over the wet cells
    double sx = 1.0 - tx, sy = 1.0 - ty;
    double w[4] = {sx * sy, tx * sy, sx * ty, tx * ty};
    double sw = 0.0, se = 0.0, su = 0.0, sv = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (h[m] > N.eps) {
        sw += w[m];
        se += w[m] * e[m];
        su += w[m] * uu[m];
        sv += w[m] * vv[m];
      }
    }
    if (sw > 0.0) {
      eta = se / sw;
      u = su / sw;
      v = sv / sw;
    } else {
      has = false;
    }
  }
  double H = 0.0;
  double bfk = fb[(size_t)fi + (size_t)fj * N.nxf];
  if (tx == 0.0 && ty == 0.0) {  // centre on a coarse centre (odd r): its depth form
    has = h[0] > N.eps;
    eta = 0.0;
    u = uu[0];
    v = vv[0];
    double dep = h[0] + (cb[k[0]] - bfk);
    if (has) H = dep > 0.0 ? dep : 0.0;
  } else if (has) {
    double dep = eta - bfk;
    H = dep > 0.0 ? dep : 0.0;
  }
  if (!(H > N.eps)) {
    u = 0.0;
    v = 0.0;
  }
  out[q] = H;
  out[N.nghost + q] = u;
  out[2 * N.nghost + q] = v;
}

// fine ghost band = lerp(G0, G1, alpha); marks the touched fused tiles
__global__ void k_ghost_apply(NestGeo N, const double* __restrict__ g0, const double* __restrict__ g1,
                              double alpha, double* __restrict__ H, double* __restrict__ U,
                              double* __restrict__ V, unsigned char* tile_prev,
                              unsigned char* tile_same, int tiles_x) {
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= N.nghost) return;
  int fi, fj;
  ghost_cell(N, q, fi, fj);
  long long G = N.nghost;
  double h = lerp(g0[q], g1[q], alpha);
  double u = lerp(g0[G + q], g1[G + q], alpha);
  double v = lerp(g0[2 * G + q], g1[2 * G + q], alpha);
  if (!(h > N.eps)) {
    u = 0.0;
    v = 0.0;
  }
  size_t k = (size_t)fi + (size_t)fj * N.nxf;
  H[k] = h;
  U[k] = u;
  V[k] = v;
  int t = fi / TBX + (fj / TBY) * tiles_x;
  tile_prev[t] = 3;
  tile_same[t] = 0;
}

// restrict_feedback: one thread per window cell
__global__ void k_restrict(NestGeo N, const double* __restrict__ fH, const double* __restrict__ fU,
                           const double* __restrict__ fV, double* __restrict__ cH,
                           double* __restrict__ cU, double* __restrict__ cV,
                           unsigned char* tile_prev, unsigned char* tile_same, int tiles_x) {
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= (long long)N.ni * N.nj) return;
  int ci = (int)(q % N.ni), cj = (int)(q / N.ni);
  double sh = 0.0, su = 0.0, sv = 0.0;
  for (int b = 0; b < N.r; ++b) {
    size_t row = (size_t)(N.gw + cj * N.r + b) * N.nxf + (size_t)(N.gw + ci * N.r);
    for (int a = 0; a < N.r; ++a) {
      sh += fH[row + a];
      su += fU[row + a];
      sv += fV[row + a];
    }
  }
  double rr = (double)(N.r * N.r);
  int i = N.i0 + ci, j = N.j0 + cj;
  size_t k = (size_t)i + (size_t)j * N.cnx;
  cH[k] = sh / rr;
  cU[k] = su / rr;
  cV[k] = sv / rr;
  int t = i / TBX + (j / TBY) * tiles_x;
  tile_prev[t] = 3;
  tile_same[t] = 0;
}

// tap_fsum += tap_f (after each fine substep, in substep order)
__global__ void k_tap_add(int n, const double* __restrict__ a, double* __restrict__ sum) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) sum[q] = sum[q] + a[q];
}

// Flux correction (refluxing): the coarse cells just outside the window lost
// or gained the coarse step's face volumes vc; the window (now the fine
// means) exchanged the fine substeps' vf instead.  Each outside cell gets
// (vc - vf) / h^2 on the inflow sides (west, south) and (vf - vc) / h^2 on
// the outflow sides, which makes the coupled system conservative; a cell
// driven below 0 is clamped (and dried).  One thread per boundary face.
__global__ void k_reflux(NestGeo N, const double* __restrict__ tc, const double* __restrict__ tf,
                         double hc, double hf, double* H, double* HUx, double* HUy,
                         unsigned char* tile_prev, unsigned char* tile_same, int tiles_x,
                         double* clampv) {
  const int nq = 2 * (N.ni + N.nj);
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int side, k, fo, i, j;
  if (q < N.nj) {
    side = 0; k = q; fo = k * N.r; i = N.i0 - 1; j = N.j0 + k;
  } else if (q < 2 * N.nj) {
    side = 1; k = q - N.nj; fo = N.r * N.nj + k * N.r; i = N.i0 + N.ni; j = N.j0 + k;
  } else if (q < 2 * N.nj + N.ni) {
    side = 2; k = q - 2 * N.nj; fo = 2 * N.r * N.nj + k * N.r; i = N.i0 + k; j = N.j0 - 1;
  } else {
    side = 3; k = q - 2 * N.nj - N.ni; fo = 2 * N.r * N.nj + N.r * N.ni + k * N.r; i = N.i0 + k;
    j = N.j0 + N.nj;
  }
  const double vc = tc[q] * hc;
  double vf = 0.0;
  for (int b = 0; b < N.r; ++b) vf = vf + tf[fo + b];
  vf = vf * hf;
  const double d = (side == 0 || side == 2) ? (vc - vf) / (hc * hc) : (vf - vc) / (hc * hc);
  const size_t c = (size_t)i + (size_t)j * N.cnx;
  double h = H[c] + d;
  // a dry-side cell cannot give what the fine side drew at a wet/dry front:
  // clamp and log the volume added, like the step's own clamp deficit
  clampv[q] = h < 0.0 ? (0.0 - h) * (hc * hc) : 0.0;
  if (!(h > 0.0)) h = 0.0;
  H[c] = h;
  if (!(h > N.eps)) {
    HUx[c] = 0.0;
    HUy[c] = 0.0;
  }
  int t = i / TBX + (j / TBY) * tiles_x;
  tile_prev[t] = 3;
  tile_same[t] = 0;
}

NestGeo nest_geo(const swf_nest* n) {
  NestGeo N;
  N.cnx = n->coarse->geo.nx;
  N.cny = n->coarse->geo.ny;
  N.i0 = n->d.i0;
  N.j0 = n->d.j0;
  N.ni = n->d.ni;
  N.nj = n->d.nj;
  N.r = n->d.r;
  N.gw = n->d.ghost;
  N.nxf = n->nxf;
  N.nyf = n->nyf;
  N.eps = n->fine->params.eps_dry;
  N.nghost = (long long)n->nghost;
  return N;
}

int nest_err(swf_nest* n, int code, const std::string& m) {
  n->err = m;
  return code;
}

int nest_cuda(swf_nest* n, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SWF_OK;
  return nest_err(n, SWF_ECUDA, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// ---- device-driven subcycling (no host round trip per fine substep) --------
// Per substep: k_sub_begin decides on the device whether the fine grid still
// lags the global time t1 (else it marks the context idle, which makes every
// remaining kernel of the batch skip), and sets alpha and dt_cap; then the
// ghost band, the fused step with dt_cap read on the device, the face taps
// and k_sub_end (the smallest fine tau).
__global__ void k_sub_begin(StepScalars* sc, double t0, double t1, double tol, int first,
                            double tau_g, double* alpha) {
  if (stopped(sc)) return;
  const double tf = sc->t;
  if (!(t1 - tf > tol)) {  // landed on t1: the remaining substeps of the batch skip
    sc->err_key = ERR_IDLE << 58;
    return;
  }
  // the first substep is capped by the global tau itself (t1 - t0 can differ
  // from it in the last bit), later ones by the remaining time
  sc->dt_cap_dev = first ? tau_g : t1 - tf;
  *alpha = (tf - t0) / (t1 - t0);
}

__global__ void k_sub_end(const StepScalars* sc, double* tau_min) {
  if (stopped(sc)) return;
  if (sc->tau < *tau_min) *tau_min = sc->tau;
}

__global__ void k_ghost_apply_dev(NestGeo N, const double* __restrict__ g0,
                                  const double* __restrict__ g1, const double* alpha,
                                  const StepScalars* sc, double* __restrict__ H,
                                  double* __restrict__ U, double* __restrict__ V,
                                  unsigned char* tile_prev, unsigned char* tile_same,
                                  int tiles_x) {
  if (stopped(sc)) return;
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= N.nghost) return;
  int fi, fj;
  ghost_cell(N, q, fi, fj);
  long long G = N.nghost;
  const double a = *alpha;
  double h = lerp(g0[q], g1[q], a);
  double u = lerp(g0[G + q], g1[G + q], a);
  double v = lerp(g0[2 * G + q], g1[2 * G + q], a);
  if (!(h > N.eps)) {
    u = 0.0;
    v = 0.0;
  }
  size_t k = (size_t)fi + (size_t)fj * N.nxf;
  H[k] = h;
  U[k] = u;
  V[k] = v;
  int t = fi / TBX + (fj / TBY) * tiles_x;
  tile_prev[t] = 3;
  tile_same[t] = 0;
}

__global__ void k_tap_add_dev(int n, const StepScalars* sc, const double* __restrict__ a,
                              double* __restrict__ sum) {
  if (stopped(sc)) return;
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) sum[q] = sum[q] + a[q];
}

double host_t(swf_ctx* c) {
  double t = 0.0;
  cudaMemcpy(&t, &c->d_sc->t, sizeof(double), cudaMemcpyDeviceToHost);
  return t;
}

}  // namespace
}  // namespace swf

using namespace swf;

extern "C" {

int swf_nest_create(swf_ctx* coarse, swf_ctx* fine, const swf_nest_desc* d, swf_nest** out) {
  if (!coarse || !fine || !d || !out) return set_err(coarse, SWF_ECONFIG, "nest: null argument");
  *out = nullptr;
  const Geo& C = coarse->geo;
  const Geo& F = fine->geo;
  auto bad = [&](const std::string& m) { return set_err(coarse, SWF_ECONFIG, "nest: " + m); };
  if (d->r < 1) return bad("refinement factor r must be >= 1");
  if (d->ghost < 1) return bad("ghost band must be >= 1 fine cell");
  if (d->ni < 1 || d->nj < 1) return bad("empty window");
  if (C.r0 != 0 || C.r1 != C.rows || F.r0 != 0 || F.r1 != F.rows)
    return bad("strip contexts cannot be nested");
  if (coarse->device != fine->device) return bad("coarse and fine contexts on different devices");
  // bilinear stencils of the ghost band stay inside the coarse grid
  int m = (d->ghost + d->r - 1) / d->r + 1;
  if (d->i0 < m || d->j0 < m || d->i0 + d->ni + m > C.nx || d->j0 + d->nj + m > C.ny)
    return bad("window must lie strictly inside the global domain (margin " + std::to_string(m) +
               " coarse cells)");
  int nxf = d->r * d->ni + 2 * d->ghost, nyf = d->r * d->nj + 2 * d->ghost;
  if (F.nx != nxf || F.ny != nyf)
    return bad("fine grid must be " + std::to_string(nxf) + "x" + std::to_string(nyf) +
               " (r*window + 2*ghost)");
  double hf = coarse->h / d->r;
  if (std::fabs(fine->h - hf) > 1e-12 * hf) return bad("fine h must equal coarse h / r");
  swf_nest* n = new swf_nest;
  n->coarse = coarse;
  n->fine = fine;
  n->d = *d;
  n->nxf = nxf;
  n->nyf = nyf;
  n->nghost = (size_t)nxf * nyf - (size_t)(d->r * d->ni) * (size_t)(d->r * d->nj);
  cudaSetDevice(coarse->device);
  cudaError_t e = cudaSuccess;
  for (int s = 0; s < 2 && e == cudaSuccess; ++s) e = cudaMalloc(&n->g[s], 3 * n->nghost * sizeof(double));
  if (e == cudaSuccess && d->two_way) {
    size_t nc = 2 * (size_t)(d->ni + d->nj), nf = (size_t)d->r * nc;
    if (coarse->taps.n >= MAX_TAPS || fine->taps.n >= MAX_TAPS) {
      swf_nest_destroy(n);
      return bad("too many nested windows on one grid (max " + std::to_string(MAX_TAPS) + ")");
    }
    e = cudaMalloc(&n->tap_c, nc * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&n->tap_f, nf * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&n->tap_fsum, nf * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&n->clampv, nc * sizeof(double));
    if (e == cudaSuccess) {
      FaceTaps& tc = coarse->taps;
      tc.i0[tc.n] = d->i0; tc.j0[tc.n] = d->j0; tc.ni[tc.n] = d->ni; tc.nj[tc.n] = d->nj;
      tc.out[tc.n++] = n->tap_c;
      FaceTaps& tf = fine->taps;
      tf.i0[tf.n] = d->ghost; tf.j0[tf.n] = d->ghost; tf.ni[tf.n] = d->r * d->ni;
      tf.nj[tf.n] = d->r * d->nj; tf.out[tf.n++] = n->tap_f;
      invalidate_graph(coarse);  // captured steps do not record the new taps
      invalidate_graph(fine);
    }
  }
  if (e != cudaSuccess) {
    int rc = cuda_check(coarse, e, "nest allocation");
    swf_nest_destroy(n);
    return rc;
  }
  *out = n;
  return SWF_OK;
}

void swf_nest_destroy(swf_nest* n) {
  if (!n) return;
  auto unreg = [](swf_ctx* c, double* p) {
    if (!c || !p) return;
    FaceTaps& t = c->taps;
    for (int q = 0; q < t.n; ++q)
      if (t.out[q] == p) {
        for (int m = q + 1; m < t.n; ++m) {
          t.i0[m - 1] = t.i0[m]; t.j0[m - 1] = t.j0[m]; t.ni[m - 1] = t.ni[m];
          t.nj[m - 1] = t.nj[m]; t.out[m - 1] = t.out[m];
        }
        --t.n;
        invalidate_graph(c);
        break;
      }
  };
  unreg(n->coarse, n->tap_c);
  unreg(n->fine, n->tap_f);
  for (double* p : n->g) cudaFree(p);
  cudaFree(n->tap_c);
  cudaFree(n->tap_f);
  cudaFree(n->tap_fsum);
  cudaFree(n->clampv);
  cudaFree(n->d_sub);
  delete n;
}

const char* swf_nest_last_error(const swf_nest* n) { return n ? n->err.c_str() : ""; }

int swf_nest_ghost_count(const swf_nest* n, size_t* count) {
  if (!n || !count) return SWF_ECONFIG;
  *count = n->nghost;
  return SWF_OK;
}

int swf_nest_prolong(swf_nest* n, int slot) {
  if (slot < 0 || slot > 1) return nest_err(n, SWF_ECONFIG, "nest: slot must be 0 or 1");
  swf_ctx* c = n->coarse;
  cudaSetDevice(c->device);
  NestGeo N = nest_geo(n);
  unsigned blocks = (unsigned)((n->nghost + 255) / 256);
  if (blocks)
    k_prolong<<<blocks, 256, 0, c->stream>>>(N, c->H[c->cur], c->HUx[c->cur], c->HUy[c->cur], c->b,
                                             n->fine->b, n->g[slot]);
  return nest_cuda(n, cudaGetLastError(), "nest prolong");
}

int swf_nest_download_ghosts(swf_nest* n, int slot, double* out) {
  if (slot < 0 || slot > 1 || !out) return nest_err(n, SWF_ECONFIG, "nest: bad ghost download");
  cudaSetDevice(n->coarse->device);
  cudaError_t e = cudaStreamSynchronize(n->coarse->stream);
  if (e == cudaSuccess)
    e = cudaMemcpy(out, n->g[slot], 3 * n->nghost * sizeof(double), cudaMemcpyDeviceToHost);
  return nest_cuda(n, e, "nest ghost download");
}

int swf_nest_apply_ghosts(swf_nest* n, double alpha) {
  swf_ctx* f = n->fine;
  cudaSetDevice(f->device);
  // the prolongations were written on the coarse stream
  cudaError_t e = cudaStreamSynchronize(n->coarse->stream);
  if (e != cudaSuccess) return nest_cuda(n, e, "nest apply (coarse sync)");
  NestGeo N = nest_geo(n);
  unsigned blocks = (unsigned)((n->nghost + 255) / 256);
  if (blocks)
    k_ghost_apply<<<blocks, 256, 0, f->stream>>>(N, n->g[0], n->g[1], alpha, f->H[f->cur],
                                                 f->HUx[f->cur], f->HUy[f->cur],
                                                 tile_act_at(f, 1 - f->cur), f->d_tile_same,
                                                 f->geo.tiles_x);
  return nest_cuda(n, cudaGetLastError(), "nest apply ghosts");
}

int swf_nest_restrict(swf_nest* n) {
  swf_ctx* c = n->coarse;
  swf_ctx* f = n->fine;
  cudaSetDevice(c->device);
  cudaError_t e = cudaStreamSynchronize(f->stream);
  if (e != cudaSuccess) return nest_cuda(n, e, "nest restrict (fine sync)");
  NestGeo N = nest_geo(n);
  long long cells = (long long)N.ni * N.nj;
  k_restrict<<<(unsigned)((cells + 255) / 256), 256, 0, c->stream>>>(
      N, f->H[f->cur], f->HUx[f->cur], f->HUy[f->cur], c->H[c->cur], c->HUx[c->cur],
      c->HUy[c->cur], tile_act_at(c, 1 - c->cur), c->d_tile_same, c->geo.tiles_x);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return nest_cuda(n, e, "nest restrict");
}

static int nest_reflux(swf_nest* n, double* clamp_volume) {
  swf_ctx* c = n->coarse;
  NestGeo N = nest_geo(n);
  int nq = 2 * (N.ni + N.nj);
  k_reflux<<<(nq + 255) / 256, 256, 0, c->stream>>>(
      N, n->tap_c, n->tap_fsum, c->h, n->fine->h, c->H[c->cur], c->HUx[c->cur], c->HUy[c->cur],
      tile_act_at(c, 1 - c->cur), c->d_tile_same, c->geo.tiles_x, n->clampv);
  cudaError_t e = cudaGetLastError();
  std::vector<double> v(nq);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(v.data(), n->clampv, nq * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  for (double x : v) *clamp_volume += x;  // face order: deterministic
  return nest_cuda(n, e, "nest reflux");
}

int swf_coupled_step(swf_ctx* coarse, swf_nest** nests, int nn, double dt_cap,
                     swf_coupled_info* info) {
  swf_coupled_info tmp{};
  swf_coupled_info& I = info ? *info : tmp;
  I = swf_coupled_info{};
  for (int q = 0; q < nn; ++q)
    if (!nests[q] || nests[q]->coarse != coarse)
      return set_err(coarse, SWF_ECONFIG, "coupled_step: nest does not belong to this grid");
  cudaSetDevice(coarse->device);
  double t0 = host_t(coarse);
  for (int q = 0; q < nn; ++q) {
    double tf = host_t(nests[q]->fine);
    if (tf != t0)
      return set_err(coarse, SWF_ECONFIG,
                     "coupled_step: nested grid not synchronized with the global grid");
    int rc = swf_nest_prolong(nests[q], 0);
    if (rc) return set_err(coarse, rc, nests[q]->err);
  }
  // the global step; its exact StepInfo volumes are reduced on the coarse
  // stream while the fine substeps run on theirs (the terms, the step's
  // block flags and its step-start depth stay put until the next global step)
  coarse->defer_volumes = 1;
  int rc = swf_step(coarse, dt_cap, &I.coarse);
  coarse->defer_volumes = 0;
  if (rc) return rc;  // global abort: both levels untouched
  double t1 = host_t(coarse);
  double tau_g = t1 - t0;
  I.tau = I.coarse.tau;
  I.fine_tau_min = INFINITY;
  // the ghosts at t1 of every window, then (behind them on the coarse
  // stream) the global step's exact volumes, overlapping the fine substeps,
  // which wait for the prolongations only
  for (int q = 0; q < nn; ++q) {
    rc = swf_nest_prolong(nests[q], 1);
    if (rc) return set_err(coarse, rc, nests[q]->err);
  }
  cudaEvent_t prolonged = nullptr;
  cudaError_t e = cudaEventCreateWithFlags(&prolonged, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(prolonged, coarse->stream);
  if (e != cudaSuccess) return cuda_check(coarse, e, "nest prolongation event");
  struct EventGuard {
    cudaEvent_t ev;
    ~EventGuard() { cudaEventDestroy(ev); }
  } guard{prolonged};
  if (coarse->mode == 0 && (rc = fused_exact_volumes(coarse))) return rc;
  for (int q = 0; q < nn; ++q) {
    swf_nest* n = nests[q];
    swf_ctx* f = n->fine;
    double tol = std::fmax(1e-9 * tau_g, 8.0 * 2.220446049250313e-16 * std::fabs(t1));
    int sub = 0;
    const int nft = n->tap_f ? 2 * n->d.r * (n->d.ni + n->d.nj) : 0;
    if (nft) cudaMemsetAsync(n->tap_fsum, 0, nft * sizeof(double), f->stream);
    // the fine substeps in device-driven batches (the prolongations of t0 and
    // t1 were written on the coarse stream): one host synchronisation per
    // batch, sized from the previous coupled step
    e = cudaStreamWaitEvent(f->stream, prolonged, 0);
    if (e != cudaSuccess) return cuda_check(coarse, e, "nest (wait for the ghosts)");
    if (!n->d_sub && (e = cudaMalloc(&n->d_sub, 2 * sizeof(double))) != cudaSuccess)
      return cuda_check(coarse, e, "nest subcycling scalars");
    const double init[2] = {0.0, INFINITY};
    cudaMemcpyAsync(n->d_sub, init, sizeof init, cudaMemcpyHostToDevice, f->stream);
    NestGeo N = nest_geo(n);
    const unsigned gblocks = (unsigned)((n->nghost + 255) / 256);
    bool landed = false;
    // batch size: the previous coupled step's substep count (capped), then
    // one substep per batch while the fine grid still lags -- an idle
    // substep costs about as much as the host round trip it saves
    int batch = std::min(32, std::max(1, n->last_subs));
    while (!landed) {
      int cur0 = f->cur;
      if ((rc = batch_reset(f))) return set_err(coarse, rc, swf_last_error(f));
      for (int b = 0; b < batch; ++b) {
        k_sub_begin<<<1, 1, 0, f->stream>>>(f->d_sc, t0, t1, tol, sub == 0 && b == 0 ? 1 : 0,
                                            I.tau, n->d_sub);
        if (gblocks)
          k_ghost_apply_dev<<<gblocks, 256, 0, f->stream>>>(
              N, n->g[0], n->g[1], n->d_sub, f->d_sc, f->H[f->cur], f->HUx[f->cur],
              f->HUy[f->cur], tile_act_at(f, 1 - f->cur), f->d_tile_same, f->geo.tiles_x);
        if ((rc = fused_enqueue_step(f, -1.0))) {  // dt_cap from k_sub_begin
          f->cur = cur0;
          return set_err(coarse, rc, std::string("nested grid: ") + swf_last_error(f));
        }
        if (nft)
          k_tap_add_dev<<<(nft + 255) / 256, 256, 0, f->stream>>>(nft, f->d_sc, n->tap_f,
                                                                  n->tap_fsum);
        k_sub_end<<<1, 1, 0, f->stream>>>(f->d_sc, n->d_sub + 1);
      }
      e = cudaStreamSynchronize(f->stream);
      if (e != cudaSuccess) return cuda_check(coarse, e, "nest substeps");
      int done = 0;
      rc = batch_commit(f, cur0, batch, &done);
      if (rc) return set_err(coarse, rc, std::string("nested grid: ") + swf_last_error(f));
      sub += done;
      // landed: marked idle, or the last substep of the batch reached t1
      landed = (f->h_sc->err_key >> 58) == ERR_IDLE || !(t1 - f->h_sc->t > tol);
      if (sub > 1000000)
        return set_err(coarse, SWF_ENUMERICAL, "nested grid: subcycling does not converge");
      batch = 1;
    }
    // the idle marker has done its job: clear it for the fine context's next calls
    f->h_sc->err_key = ERR_NONE;
    e = cudaMemcpyAsync(&f->d_sc->err_key, &f->h_sc->err_key, sizeof(unsigned long long),
                        cudaMemcpyHostToDevice, f->stream);
    if (e != cudaSuccess) return cuda_check(coarse, e, "nest idle reset");
    n->last_subs = sub;
    double sub_scalars[2];
    e = cudaMemcpy(sub_scalars, n->d_sub, sizeof sub_scalars, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_check(coarse, e, "nest substep taus");
    if (sub_scalars[1] < I.fine_tau_min) I.fine_tau_min = sub_scalars[1];
    // land exactly on the global time
    e = cudaMemcpy(&f->d_sc->t, &t1, sizeof(double), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_check(coarse, e, "nest time sync");
    f->h_t = t1;
    I.substeps_total += sub;
    if (sub > I.substeps_max) I.substeps_max = sub;
    if (n->d.two_way) {
      rc = swf_nest_restrict(n);
      if (rc) return set_err(coarse, rc, n->err);
      rc = nest_reflux(n, &I.reflux_clamp_volume);
      if (rc) return set_err(coarse, rc, n->err);
    }
  }
  if (nn == 0) I.fine_tau_min = 0.0;
  // the global step's volumes (fused path: reduced behind the substeps)
  if (coarse->mode == 0) {
    double vol[3];
    cudaError_t ev = cudaStreamSynchronize(coarse->stream);
    if (ev == cudaSuccess)
      ev = cudaMemcpy(vol, &coarse->d_sc->deficit, sizeof vol, cudaMemcpyDeviceToHost);
    if (ev != cudaSuccess) return cuda_check(coarse, ev, "coupled step volumes");
    I.coarse.clamp_deficit_volume = vol[0];
    I.coarse.source_volume = vol[1];
    I.coarse.boundary_outflow_volume = vol[2];
  }
  return SWF_OK;
}

}  // extern "C"
