// swf_capi.cu — the C ABI of include/swf.h: context lifecycle, validation
// with the reference's error convention, state transfer, the step entry
// points, CUDA-graph replay for batched runs, and device-side KAT helpers.
//
// Validation messages and order follow the reference constructor and setters
// (grid.cpp:13-21, 42-51, 77-82; sources.cpp:22-33; stepper.cpp:31-37,
// 127-170).  There is no CPU fallback: every compute entry point launches
// sm_100a kernels and fails with SWF_ECUDA when no device is usable.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "swf_internal.cuh"

namespace swf {

static thread_local std::string g_err;

int set_err(swf_ctx* c, int code, const std::string& msg) {
  (c ? c->err : g_err) = msg;
  return code;
}

int cuda_check(swf_ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SWF_OK;
  return set_err(c, SWF_ECUDA, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

size_t local_cells(const swf_ctx* c) { return (size_t)c->geo.nx * (size_t)c->geo.rows; }

void invalidate_mask(swf_ctx* c) {
  if (!c->d_sc) return;
  cudaMemsetAsync(&c->d_sc->mask_valid, 0, sizeof(int), c->stream);
  // a host step that failed before k_tau may have left mask_fresh set: the
  // flags it refers to do not describe a newly uploaded state
  cudaMemsetAsync(&c->d_sc->mask_fresh, 0, sizeof(int), c->stream);
}

void fill_block_counts(const swf_ctx* c, const StepScalars* sc, swf_step_info* info) {
  int total = c->geo.nbx * (c->geo.bj1 - c->geo.bj0);
  info->total_blocks = total;
  info->lagrangian_blocks = c->geo.skip ? sc->lag_act : total;
  info->flux_blocks = c->geo.skip ? sc->flux_act : total;
  // active_fraction, block.cpp:81-87 (mask-based, independent of skipping)
  info->active_fraction = total ? static_cast<double>(sc->flux_act) / total : 0.0;
}

int check_device_error(swf_ctx* c) {
  cudaError_t e = cudaMemcpy(c->h_sc, c->d_sc, sizeof(StepScalars), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_check(c, e, "scalar readback");
  unsigned long long key = c->h_sc->err_key;
  if (key == ERR_NONE || (key >> 58) == ERR_IDLE) return SWF_OK;
  unsigned long long kind = key >> 58;
  const Geo& G = c->geo;
  if (kind == ERR_DT) {
    // stepper.cpp:259-262 (std::to_string formats with %f; a speed near
    // DBL_MAX prints ~310 digits, so the text is sized, not truncated)
    const char* fmt = "timestep %f s fell below the abort floor %f s (max wave speed %f m/s)";
    const double* v = c->h_sc->err_val;
    std::string buf((size_t)snprintf(nullptr, 0, fmt, v[0], v[1], v[2]) + 1, '\0');
    snprintf(&buf[0], buf.size(), fmt, v[0], v[1], v[2]);
    buf.pop_back();
    return set_err(c, SWF_ENUMERICAL, buf);
  }
  if (kind == ERR_PEER)
    return set_err(c, SWF_ENUMERICAL, "strip stopped: another strip of the group aborted the step");
  unsigned long long ib = (key >> 24) & ((1ull << 34) - 1);
  unsigned long long low = key & ((1ull << 24) - 1);
  int bi = (int)(ib % G.nbx), bj = (int)(ib / G.nbx);
  int i0 = bi * G.bs, j0 = bj * G.bs;
  if (kind == ERR_CFL) {
    int i = i0 + (int)(low % G.bs), j = j0 + (int)(low / G.bs);
    char buf[256];
    snprintf(buf, sizeof buf,
             "particle displacement reached h/2 at cell (%d,%d); the Courant number is too large "
             "for this flow",
             i, j);
    return set_err(c, SWF_ENUMERICAL, buf);
  }
  // ERR_FLUX: decode the face that the reference's serial traversal reports
  long long p = (long long)((1ull << 24) - 1 - low);
  long long span = G.bs + 2, ss = span * span;
  int rank = (int)(p / (2 * ss));
  long long within = p % (2 * ss);
  int ei0 = i0 - (rank == 1 ? G.bs : 0), ej0 = j0 - (rank == 0 ? G.bs : 0);
  int ci, cj;
  if (within < ss) {  // x face: a = row, f = iface; ka = (f-1, a)
    int a = ej0 + (int)(within / span), f = ei0 + (int)(within % span);
    ci = f - 1;
    cj = a;
  } else {  // y face: a = column, f = jface; ka = (a, f-1)
    long long w2 = within - ss;
    int a = ei0 + (int)(w2 / span), f = ej0 + (int)(w2 % span);
    ci = a;
    cj = f - 1;
  }
  char buf[128];
  snprintf(buf, sizeof buf, "non-finite flux near cell (%d,%d)", ci, cj);
  return set_err(c, SWF_ENUMERICAL, buf);
}

size_t fused_tile_bytes();

}  // namespace swf

using namespace swf;

namespace {

int validate_control(swf_ctx* c, const swf_control* k) {
  if (!(k->courant > 0.0 && k->courant < 1.0))
    return set_err(c, SWF_ECONFIG, "timestep: Courant number must be in (0,1)");
  if (!(k->dt_max > 0.0)) return set_err(c, SWF_ECONFIG, "timestep: dt_max must be positive");
  if (!(k->dt_min > 0.0 && k->dt_min < k->dt_max))
    return set_err(c, SWF_ECONFIG, "timestep: need 0 < dt_min < dt_max");
  return SWF_OK;
}

int validate_setup(const swf_terrain* T, const swf_params* P, size_t n) {
  if (T->nx < 1 || T->ny < 1) return set_err(nullptr, SWF_ECONFIG, "terrain: nx and ny must be >= 1");
  if (!(T->h > 0.0)) return set_err(nullptr, SWF_ECONFIG, "terrain: cell size must be positive");
  if (!T->b) return set_err(nullptr, SWF_ECONFIG, "terrain: bed array size mismatch");
  if ((long long)T->nx * T->ny > 2147483647LL)
    return set_err(nullptr, SWF_ECONFIG, "terrain: more than 2^31-1 cells");
  for (size_t k = 0; k < n; ++k)
    if (!std::isfinite(T->b[k]))
      return set_err(nullptr, SWF_ECONFIG,
                     "terrain: non-finite bed elevation at cell " + std::to_string(k));
  if (!(P->g > 0.0)) return set_err(nullptr, SWF_ECONFIG, "params: gravity must be positive");
  if (P->n_manning < 0.0) return set_err(nullptr, SWF_ECONFIG, "params: Manning coefficient must be >= 0");
  if (P->n_field)
    for (size_t k = 0; k < n; ++k)
      if (P->n_field[k] < 0.0) return set_err(nullptr, SWF_ECONFIG, "params: Manning field must be >= 0");
  if (P->nu < 0.0) return set_err(nullptr, SWF_ECONFIG, "params: viscosity must be >= 0");
  if (!(P->rho_water > 0.0)) return set_err(nullptr, SWF_ECONFIG, "params: water density must be positive");
  if (P->rho_air < 0.0) return set_err(nullptr, SWF_ECONFIG, "params: air density must be >= 0");
  if (!(P->eps_dry > 0.0)) return set_err(nullptr, SWF_ECONFIG, "params: dry threshold must be positive");
  return SWF_OK;
}

void drop_graph(swf_ctx* c) {
  if (c->graph) cudaGraphExecDestroy(c->graph);
  c->graph = nullptr;
  c->graph_dt_cap = -1.0;
}

// geometry derived from options (block size, boundaries, skipping)
int apply_options(swf_ctx* c, const swf_options* o) {
  if (o->block_size < 1) return set_err(c, SWF_ECONFIG, "stepper: block size must be >= 1");
  Geo& G = c->geo;
  int old_bs = G.bs, old_bj0 = G.bj0, old_bj1 = G.bj1;
  c->opt = *o;
  if (c->opt.workers < 1) c->opt.workers = 1;
  G.bs = o->block_size;
  G.nbx = (G.nx + G.bs - 1) / G.bs;
  G.nby = (G.ny + G.bs - 1) / G.bs;
  int jglo = G.jg0 + G.r0, jghi = G.jg0 + G.r1;  // owned global rows
  if (jglo % G.bs != 0 || (jghi % G.bs != 0 && jghi != G.ny))
    return set_err(c, SWF_ECONFIG, "strip boundaries must be multiples of the block size");
  G.bj0 = jglo / G.bs;
  G.bj1 = (jghi + G.bs - 1) / G.bs;
  G.west_refl = o->west == SWF_EDGE_REFLECTIVE;
  G.east_refl = o->east == SWF_EDGE_REFLECTIVE;
  G.south_refl = o->south == SWF_EDGE_REFLECTIVE;
  G.north_refl = o->north == SWF_EDGE_REFLECTIVE;
  G.skip = o->skip_dry_blocks != 0;
  if (!c->d_interior || old_bs != G.bs || old_bj0 != G.bj0 || old_bj1 != G.bj1) {
    cudaFree(c->d_interior);
    cudaFree(c->d_halo);
    cudaFree(c->d_bflag);
    size_t nb = (size_t)G.nbx * (G.bj1 - G.bj0);
    cudaError_t e = cudaMalloc(&c->d_interior, (nb ? nb : 1) * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_halo, (nb ? nb : 1) * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_bflag, nb ? nb : 1);
    if (e == cudaSuccess) e = cudaMemset(c->d_interior, 0, (nb ? nb : 1) * sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->d_halo, 0, (nb ? nb : 1) * sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->d_bflag, 0, nb ? nb : 1);
    if (e != cudaSuccess) return cuda_check(c, e, "mask allocation");
  }
  drop_graph(c);
  return SWF_OK;
}

void apply_control(swf_ctx* c, const swf_control* k) {
  c->ctl = *k;
  c->geo.courant = k->courant;
  c->geo.dt_max = k->dt_max;
  c->geo.dt_min = k->dt_min;
  drop_graph(c);
}

int create_impl(const swf_terrain* T, const swf_params* P, const swf_control* K,
                const swf_options* O, int j0, int j1, int device, swf_ctx** out) {
  *out = nullptr;
  if (!T || !P || !K || !O) return set_err(nullptr, SWF_ECONFIG, "null argument");
  if (T->ny >= 1 && (j0 < 0 || j1 > T->ny || j0 >= j1))
    return set_err(nullptr, SWF_ECONFIG, "strip rows out of range");
  // a neighbour's SWF_HALO ghost rows are this strip's owned boundary rows
  if (T->ny >= 1 && (j0 > 0 || j1 < T->ny) && j1 - j0 < SWF_HALO)
    return set_err(nullptr, SWF_ECONFIG,
                   "strip: a strip with a neighbour must own at least 3 rows (the halo depth)");
  // host arrays cover the local window: global rows [j0 - glo, j1 + ghi)
  int glo = j0 > 0 ? SWF_HALO : 0, ghi = j1 < T->ny ? SWF_HALO : 0;
  if (j0 - glo < 0) glo = j0;
  if (j1 + ghi > T->ny) ghi = T->ny - j1;
  int rc = validate_setup(T, P, (size_t)(T->nx > 0 ? T->nx : 0) * (size_t)((j1 - j0) + glo + ghi));
  if (rc) return rc;
  rc = validate_control(nullptr, K);
  if (rc) return rc;
  if (O->block_size < 1) return set_err(nullptr, SWF_ECONFIG, "stepper: block size must be >= 1");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return set_err(nullptr, SWF_ECUDA,
                   std::string("no CUDA device available (libswflood_cuda has no CPU path): ") +
                       cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return set_err(nullptr, SWF_ECONFIG, "device index out of range");
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_check(nullptr, e, "cudaSetDevice");

  swf_ctx* c = new swf_ctx();
  c->device = device;
  c->h = T->h;
  c->x0 = T->x0;
  c->y0 = T->y0;
  c->params = *P;
  c->params.n_field = nullptr;
  Geo& G = c->geo;
  G.nx = T->nx;
  G.ny = T->ny;
  G.jg0 = j0 - glo;
  G.rows = (j1 - j0) + glo + ghi;
  G.r0 = glo;
  G.r1 = glo + (j1 - j0);
  G.has_nfield = P->n_field != nullptr;
  G.n_manning = P->n_manning;
  G.P.g = P->g;
  G.P.nu = P->nu;
  G.P.omega_z = P->omega_z;
  G.P.c_a = P->c_a;
  G.P.rho_air = P->rho_air;
  G.P.rho_water = P->rho_water;
  G.P.eps = P->eps_dry;
  G.P.h = T->h;
  G.P.inv_h2 = 1.0 / (T->h * T->h);
  G.P.two_h = 2.0 * T->h;
  // divisors of eta_grad_comp; r = 0 makes rdiv use plain division until a
  // kernel refines the reciprocal on the device (with_recips)
  G.P.rh.b = T->h;
  G.P.rh.r = 0.0;
  G.P.r2h.b = G.P.two_h;
  G.P.r2h.r = 0.0;
  G.tiles_x = (G.nx + 31) / 32;
  G.tiles_y = (G.r1 - G.r0 + 15) / 16;
  apply_control(c, K);
  rc = apply_options(c, O);
  if (rc) {
    g_err = c->err;
    swf_destroy(c);
    return rc;
  }
  size_t n = local_cells(c);
  size_t bytes = n * sizeof(double);
  const double* bsrc = T->b;  // window rows [jg0, jg0 + rows)
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&c->b, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(c->b, bsrc, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && P->n_field) {
    e = cudaMalloc(&c->nf, bytes);
    if (e == cudaSuccess)
      e = cudaMemcpy(c->nf, P->n_field, bytes, cudaMemcpyHostToDevice);
  }
  for (int s = 0; s < 2 && e == cudaSuccess; ++s) {
    e = cudaMalloc(&c->H[s], bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->HUx[s], bytes);
    if (e == cudaSuccess) e = cudaMalloc(&c->HUy[s], bytes);
    if (e == cudaSuccess) e = cudaMemset(c->H[s], 0, bytes);
    if (e == cudaSuccess) e = cudaMemset(c->HUx[s], 0, bytes);
    if (e == cudaSuccess) e = cudaMemset(c->HUy[s], 0, bytes);
  }
  // f' is written for wet cells only, but k_step stages it for its whole
  // region (and discards it for dry cells): start from defined values
  if (e == cudaSuccess) e = cudaMalloc(&c->fpx, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->fpy, bytes);
  if (e == cudaSuccess) e = cudaMemset(c->fpx, 0, bytes);
  if (e == cudaSuccess) e = cudaMemset(c->fpy, 0, bytes);
  size_t nt = (size_t)G.tiles_x * G.tiles_y;
  if (e == cudaSuccess) e = cudaMalloc(&c->d_tile_act, 2 * (nt ? nt : 1));
  if (e == cudaSuccess) e = cudaMemset(c->d_tile_act, 0, 2 * (nt ? nt : 1));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_tile_same, nt ? nt : 1);
  if (e == cudaSuccess) e = cudaMemset(c->d_tile_same, 1, nt ? nt : 1);  // both buffers zero
  // per-tile diagnostic partials, then the k_reduce partials
  if (e == cudaSuccess)
    e = cudaMalloc(&c->d_part, 5 * ((nt ? nt : 1) + (size_t)fused_reduce_ctas()) * sizeof(double));
  if (e == cudaSuccess)
    e = cudaMemset(c->d_part, 0, 5 * ((nt ? nt : 1) + (size_t)fused_reduce_ctas()) * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_sig, 2 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_sc, sizeof(StepScalars));
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_sc, sizeof(StepScalars));
  if (e == cudaSuccess) {
    std::memset(c->h_sc, 0, sizeof(StepScalars));
    c->h_sc->err_key = ERR_NONE;
    c->h_sc->fail_step = -1;
    e = cudaMemcpy(c->d_sc, c->h_sc, sizeof(StepScalars), cudaMemcpyHostToDevice);
  }
  for (int i = 0; i < 10 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev[i]);
  if (e == cudaSuccess && fused_prepare(c) != SWF_OK) {
    // fused_prepare recorded the CUDA error text (out of memory, ...)
    g_err = c->err;
    swf_destroy(c);
    return SWF_ECUDA;
  }
  if (e == cudaSuccess && fused_tile_srcm(c) != SWF_OK) e = cudaErrorInvalidValue;
  if (e != cudaSuccess) {
    rc = cuda_check(nullptr, e, "context allocation");
    swf_destroy(c);
    return rc;
  }
  *out = c;
  return SWF_OK;
}

// reset the device error/step counters before a new batch
int reset_counters(swf_ctx* c) {
  c->h_sc->err_key = ERR_NONE;
  c->h_sc->fail_step = -1;
  c->h_sc->steps_done = 0;
  cudaError_t e = cudaMemcpyAsync(&c->d_sc->err_key, &c->h_sc->err_key, sizeof(unsigned long long),
                                  cudaMemcpyHostToDevice, c->stream);
  int zero = 0, neg = -1;
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&c->d_sc->steps_done, &zero, sizeof(int), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&c->d_sc->fail_step, &neg, sizeof(int), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return cuda_check(c, e, "counter reset");
}

void fill_fused_info(swf_ctx* c, swf_step_info* info) {
  const StepScalars* s = c->h_sc;
  std::memset(info, 0, sizeof *info);
  info->tau = s->tau;
  fill_block_counts(c, s, info);
  info->clamp_deficit_volume = s->deficit;
  info->source_volume = s->srcvol;
  info->boundary_outflow_volume = s->outflow;
  if (c->timing) {
    float ms;
    // buckets: mask (begin+K1), forces (K2), dt (K3 tail), flux (K4..K8 fused), finalize
    int map[5][2] = {{0, 0}, {1, 1}, {2, 2}, {3, 6}, {4, 7}};
    const cudaEvent_t* E = c->ev;
    if (c->tslots > 0 && c->tstep > 0) E = &c->tev[(size_t)((c->tstep - 1) % c->tslots) * 6];
    for (auto& m : map) {
      if (cudaEventElapsedTime(&ms, E[m[0]], E[m[0] + 1]) == cudaSuccess)
        info->timings[m[1]] = ms * 1e-3;
    }
  }
}

// After a synchronised batch: roll back the ping-pong index to the last
// committed state and report the device error, if any.
int commit_batch(swf_ctx* c, int cur_start, int enqueued, int* done) {
  int rc = check_device_error(c);
  int ok = c->h_sc->steps_done;
  if (done) *done = ok;
  (void)enqueued;
  c->cur = (cur_start + ok) & 1;
  c->h_t = c->h_sc->t;
  return rc;
}

}  // namespace

namespace swf {
void invalidate_graph(swf_ctx* c) { drop_graph(c); }
int batch_reset(swf_ctx* c) { return reset_counters(c); }
int batch_commit(swf_ctx* c, int cur_start, int enqueued, int* done) {
  return commit_batch(c, cur_start, enqueued, done);
}
}  // namespace swf

extern "C" {

int swf_create(const swf_terrain* terrain, const swf_params* params, const swf_control* control,
               const swf_options* options, swf_ctx** out) {
  if (!out) return set_err(nullptr, SWF_ECONFIG, "null output pointer");
  return create_impl(terrain, params, control, options, 0, terrain ? terrain->ny : 0, 0, out);
}

int swf_create_strip(const swf_terrain* terrain, const swf_params* params,
                     const swf_control* control, const swf_options* options, int j0, int j1,
                     int device, swf_ctx** out) {
  if (!out) return set_err(nullptr, SWF_ECONFIG, "null output pointer");
  return create_impl(terrain, params, control, options, j0, j1, device, out);
}

void swf_destroy(swf_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graph(c);
  stage_free(c);
  void* ptrs[] = {c->b, c->nf, c->H[0], c->H[1], c->HUx[0], c->HUx[1], c->HUy[0], c->HUy[1],
                  c->fpx, c->fpy, c->d_src, c->d_ht, c->d_hq, c->d_sig, c->d_wt, c->d_wv,
                  c->d_interior, c->d_halo, c->d_bflag, c->d_tile_act, c->d_tile_same,
                  c->d_tile_srcm, c->d_redo_f, c->d_redo_s, c->d_list_f, c->d_list_s,
                  c->d_part, c->d_sc, c->d_redo_l, c->d_half[0], c->d_half[1], c->d_half[2],
                  c->d_xdef, c->d_xsrc, c->d_xbpart, c->d_xface, c->d_lamn, c->d_gxy};
  for (void* p : ptrs) cudaFree(p);
  if (c->h_sc) cudaFreeHost(c->h_sc);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->tev) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* swf_last_error(const swf_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

int swf_set_wind(swf_ctx* c, int n, const double* t, const double* wx, const double* wy) {
  for (int k = 1; k < n; ++k)
    if (!(t[k] > t[k - 1])) return set_err(c, SWF_ECONFIG, "wind: sample times must be strictly increasing");
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  c->h_wt.assign(t, t + n);
  c->h_wv.resize(2 * (size_t)n);
  for (int k = 0; k < n; ++k) {
    c->h_wv[2 * k] = wx[k];
    c->h_wv[2 * k + 1] = wy[k];
  }
  cudaFree(c->d_wt);
  cudaFree(c->d_wv);
  c->d_wt = c->d_wv = nullptr;
  cudaError_t e = cudaSuccess;
  if (n > 0) {
    e = cudaMalloc(&c->d_wt, n * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_wv, 2 * n * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(c->d_wt, t, n * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(c->d_wv, c->h_wv.data(), 2 * n * sizeof(double), cudaMemcpyHostToDevice);
  }
  c->geo.nwind = n;
  drop_graph(c);
  return cuda_check(c, e, "set_wind");
}

int swf_set_sources(swf_ctx* c, int n, const swf_source* s) {
  const Geo& G = c->geo;
  for (int k = 0; k < n; ++k) {
    std::string nm = "source 'src" + std::to_string(k) + "': ";
    if (s[k].i0 > s[k].i1 || s[k].j0 > s[k].j1) return set_err(c, SWF_ECONFIG, nm + "empty cell rectangle");
    bool in0 = s[k].i0 >= 0 && s[k].i0 < G.nx && s[k].j0 >= 0 && s[k].j0 < G.ny;
    bool in1 = s[k].i1 >= 0 && s[k].i1 < G.nx && s[k].j1 >= 0 && s[k].j1 < G.ny;
    if (!in0 || !in1) return set_err(c, SWF_ECONFIG, nm + "cells outside grid");
    for (int m = 1; m < s[k].n_hydro; ++m)
      if (!(s[k].hydro_t[m] > s[k].hydro_t[m - 1]))
        return set_err(c, SWF_ECONFIG, nm + "hydrograph times must be strictly increasing");
    if (s[k].kind == SWF_SOURCE_DISCHARGE && s[k].n_hydro <= 0)
      return set_err(c, SWF_ECONFIG, nm + "discharge source needs a hydrograph");
  }
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  c->h_src.clear();
  c->h_ht.clear();
  c->h_hq.clear();
  for (int k = 0; k < n; ++k) {
    DevSrc d;
    d.kind = s[k].kind;
    d.i0 = s[k].i0;
    d.j0 = s[k].j0;
    d.i1 = s[k].i1;
    d.j1 = s[k].j1;
    d.nh = s[k].n_hydro;
    d.off = (int)c->h_ht.size();
    d.rate = s[k].rate;
    d.vx = s[k].vx;
    d.vy = s[k].vy;
    int count = (d.i1 - d.i0 + 1) * (d.j1 - d.j0 + 1);
    d.count_area = (double)count * (c->h * c->h);
    for (int m = 0; m < d.nh; ++m) {
      c->h_ht.push_back(s[k].hydro_t[m]);
      c->h_hq.push_back(s[k].hydro_q[m]);
    }
    c->h_src.push_back(d);
  }
  cudaFree(c->d_src);
  cudaFree(c->d_ht);
  cudaFree(c->d_hq);
  cudaFree(c->d_sig);
  c->d_src = nullptr;
  c->d_ht = c->d_hq = c->d_sig = nullptr;
  cudaError_t e = cudaMalloc(&c->d_sig, 2 * (n > 0 ? n : 1) * sizeof(double));
  if (e == cudaSuccess && n > 0) {
    e = cudaMalloc(&c->d_src, n * sizeof(DevSrc));
    if (e == cudaSuccess)
      e = cudaMemcpy(c->d_src, c->h_src.data(), n * sizeof(DevSrc), cudaMemcpyHostToDevice);
    size_t nh = c->h_ht.size();
    if (nh > 0) {
      if (e == cudaSuccess) e = cudaMalloc(&c->d_ht, nh * sizeof(double));
      if (e == cudaSuccess) e = cudaMalloc(&c->d_hq, nh * sizeof(double));
      if (e == cudaSuccess)
        e = cudaMemcpy(c->d_ht, c->h_ht.data(), nh * sizeof(double), cudaMemcpyHostToDevice);
      if (e == cudaSuccess)
        e = cudaMemcpy(c->d_hq, c->h_hq.data(), nh * sizeof(double), cudaMemcpyHostToDevice);
    }
  }
  c->geo.nsrc = n;
  if (e == cudaSuccess) {
    int rc = fused_tile_srcm(c);
    if (rc) return rc;
  }
  if (n == 0) stage_clear_sources(c);  // src_.clear_values(), stepper.cpp:169
  invalidate_mask(c);
  drop_graph(c);
  return cuda_check(c, e, "set_sources");
}

int swf_set_control(swf_ctx* c, const swf_control* k) {
  // control() is a plain mutable reference in the reference (stepper.hpp:100)
  apply_control(c, k);
  return SWF_OK;
}

int swf_get_control(const swf_ctx* c, swf_control* k) {
  *k = c->ctl;
  return SWF_OK;
}

int swf_set_options(swf_ctx* c, const swf_options* o) {
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  invalidate_mask(c);
  return apply_options(c, o);
}

int swf_get_options(const swf_ctx* c, swf_options* o) {
  *o = c->opt;
  return SWF_OK;
}

int swf_upload_state(swf_ctx* c, const double* H, const double* HUx, const double* HUy, double t) {
  c->state_partial = 0;
  c->mirror_valid = 0;
  cudaSetDevice(c->device);
  size_t n = local_cells(c), bytes = n * sizeof(double);
  size_t off = 0;  // host arrays cover the local window
  cudaError_t e = cudaMemcpyAsync(c->H[c->cur], H + off, bytes, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(c->HUx[c->cur], HUx + off, bytes, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(c->HUy[c->cur], HUy + off, bytes, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&c->d_sc->t, &t, sizeof(double), cudaMemcpyHostToDevice, c->stream);
  size_t nt = (size_t)c->geo.tiles_x * c->geo.tiles_y;
  if (e == cudaSuccess && nt) e = cudaMemsetAsync(c->d_tile_same, 0, nt, c->stream);
  if (e == cudaSuccess) invalidate_mask(c);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  c->h_t = t;
  return cuda_check(c, e, "upload_state");
}

int swf_download_state(swf_ctx* c, double* H, double* HUx, double* HUy, double* t) {
  if (c->state_partial)
    return set_err(c, SWF_ECONFIG,
                   "the device state is incomplete after a pinned host-buffer step (sparse "
                   "momentum ingest); upload a state first");
  cudaSetDevice(c->device);
  const Geo& G = c->geo;
  size_t off = (size_t)G.r0 * G.nx, n = (size_t)(G.r1 - G.r0) * G.nx, bytes = n * sizeof(double);
  size_t hoff = off;  // owned rows at their window position
  cudaError_t e = cudaMemcpyAsync(H + hoff, c->H[c->cur] + off, bytes, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(HUx + hoff, c->HUx[c->cur] + off, bytes, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(HUy + hoff, c->HUy[c->cur] + off, bytes, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess && t) e = cudaMemcpyAsync(t, &c->d_sc->t, sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return cuda_check(c, e, "download_state");
}

int swf_device_state(swf_ctx* c, double** H, double** HUx, double** HUy) {
  if (H) *H = c->H[c->cur];
  if (HUx) *HUx = c->HUx[c->cur];
  if (HUy) *HUy = c->HUy[c->cur];
  return SWF_OK;
}

int swf_step(swf_ctx* c, double dt_cap, swf_step_info* info) {
  if (!c->wt_host[0]) c->mirror_valid = 0;  // a resident step: the host arrays fall behind
  if (c->state_partial)
    return set_err(c, SWF_ECONFIG,
                   "the device state is incomplete after a pinned host-buffer step (sparse "
                   "momentum ingest); upload a state first");
  cudaSetDevice(c->device);
  c->last_staged = c->mode == 1;
  if (c->mode == 1) {
    int rc = reset_counters(c);
    if (rc) return rc;
    swf_step_info tmp;
    return stage_step(c, dt_cap, info ? info : &tmp);
  }
  int cur0 = c->cur;
  int rc = reset_counters(c);
  if (rc) return rc;
  rc = fused_enqueue_step(c, dt_cap);
  if (rc) {
    c->cur = cur0;
    return rc;
  }
  if (!info) return SWF_OK;  // errors surface at the next synchronising call
  if (!c->defer_volumes && (rc = fused_exact_volumes(c))) return rc;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "step");
  rc = commit_batch(c, cur0, 1, nullptr);
  if (rc) return rc;
  fill_fused_info(c, info);
  return SWF_OK;
}

int swf_step_host(swf_ctx* c, double* H, double* HUx, double* HUy, double* t, double dt_cap,
                  swf_step_info* info) {
  NvtxRange nv("swf_step_host");
  auto pinned = [](const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return a.type == cudaMemoryTypeHost && a.devicePointer == p;
  };
  cudaSetDevice(c->device);
  const bool zc = c->mode == 0 && c->geo.r0 == 0 && c->geo.r1 == c->geo.rows && pinned(H) &&
                  pinned(HUx) && pinned(HUy);
  int rc;
  if (zc && c->host_mirror) {
    // Opt-in host mirror: the caller's arrays are the device state as of the
    // last host step (same arrays, same t, no other state change since): no
    // ingest at all; otherwise one full upload re-establishes the mirror.
    // Either way k_step writes every updated cell into the arrays.
    const bool same = c->mirror_valid && c->mirror_ptr[0] == H && c->mirror_ptr[1] == HUx &&
                      c->mirror_ptr[2] == HUy && c->mirror_t == *t;
    c->mirror_valid = 0;
    if (!same) {
      rc = swf_upload_state(c, H, HUx, HUy, *t);
      if (rc) return rc;
      c->last_ingest_bytes = 3LL * 8 * (long long)local_cells(c);
    } else {
      c->last_ingest_bytes = 0;
    }
    c->wt_host[0] = H;
    c->wt_host[1] = HUx;
    c->wt_host[2] = HUy;
    swf_step_info tmp;
    rc = swf_step(c, dt_cap, info ? info : &tmp);
    c->wt_host[0] = c->wt_host[1] = c->wt_host[2] = nullptr;
    if (rc) {
      if (rc == SWF_ENUMERICAL && !fused_restore_host(c, H, HUx, HUy)) {
        cudaError_t e2 = cudaStreamSynchronize(c->stream);
        if (e2 != cudaSuccess) return cuda_check(c, e2, "step_host restore");
        // the arrays hold the step-start state again, which the device keeps
        c->mirror_valid = 1;
        c->mirror_ptr[0] = H;
        c->mirror_ptr[1] = HUx;
        c->mirror_ptr[2] = HUy;
        c->mirror_t = *t;
      }
      return rc;
    }
    cudaError_t e = cudaMemcpyAsync(t, &c->d_sc->t, sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cuda_check(c, e, "step_host write-back");
    c->mirror_valid = 1;
    c->mirror_ptr[0] = H;
    c->mirror_ptr[1] = HUx;
    c->mirror_ptr[2] = HUy;
    c->mirror_t = *t;
    return SWF_OK;
  }
  if (zc) {
    // Pinned (device-mapped) arrays: the depth is copied in full by the copy
    // engine, the block mask computed from it, and the momentum read over
    // PCIe for the flux-active tiles only (fused_ingest_hu); the result goes
    // back the same way, tile by tile, after the step committed.
    size_t n = local_cells(c), bytes = n * sizeof(double);
    rc = reset_counters(c);
    if (rc) return rc;
    cudaError_t e = cudaMemcpyAsync(c->H[c->cur], H, bytes, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(&c->d_sc->t, t, sizeof(double), cudaMemcpyHostToDevice, c->stream);
    size_t nt = (size_t)c->geo.tiles_x * c->geo.tiles_y;
    if (e == cudaSuccess && nt) e = cudaMemsetAsync(c->d_tile_same, 0, nt, c->stream);
    if (e != cudaSuccess) return cuda_check(c, e, "step_host ingest");
    invalidate_mask(c);
    if ((rc = launch_begin(c, dt_cap)) || (rc = launch_mask(c)) || (rc = fused_ingest_hu(c, HUx, HUy)))
      return rc;
    // the tile flags now describe this state: the forces phase visits only
    // tiles with a wet cell in their blocks or rings (k_flist)
    e = cudaMemsetAsync(&c->d_sc->mask_fresh, 1, sizeof(int), c->stream);
    if (e != cudaSuccess) return cuda_check(c, e, "step_host mask");
    c->state_partial = 0;
    // k_step writes each updated cell into the caller's arrays as it goes
    // (PCIe writes overlapped with the step's arithmetic)
    c->wt_host[0] = H;
    c->wt_host[1] = HUx;
    c->wt_host[2] = HUy;
    swf_step_info tmp;
    rc = swf_step(c, dt_cap, info ? info : &tmp);
    c->wt_host[0] = c->wt_host[1] = c->wt_host[2] = nullptr;
    c->state_partial = 1;
    if (rc) {
      // numerical abort: put the step-start values back where the step may
      // have written (state untouched, stepper.cpp:391-399, 568-577)
      if (rc == SWF_ENUMERICAL) {
        int rr = fused_restore_host(c, H, HUx, HUy);
        if (!rr) {
          cudaError_t e2 = cudaStreamSynchronize(c->stream);
          if (e2 != cudaSuccess) return cuda_check(c, e2, "step_host restore");
        }
      }
      return rc;
    }
    int na = 0, ntot = 0, cpt = 0;
    swf_active_tiles(c, &na, &ntot, &cpt);
    c->last_ingest_bytes = (long long)bytes + 2LL * 8 * na * cpt;
    e = cudaMemcpyAsync(t, &c->d_sc->t, sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    return cuda_check(c, e, "step_host write-back");
  }
  rc = swf_upload_state(c, H, HUx, HUy, *t);
  if (rc) return rc;
  c->last_ingest_bytes = 3LL * 8 * (long long)local_cells(c);
  swf_step_info tmp;
  rc = swf_step(c, dt_cap, info ? info : &tmp);
  if (rc) return rc;
  return swf_download_state(c, H, HUx, HUy, t);
}

const char* swf_build_flavor(void) { return SWF_FAST ? "fast" : "exact"; }

int swf_last_writeback_bytes(swf_ctx* c, long long* bytes) {
  if (!c || !bytes) return SWF_ECONFIG;
  *bytes = 8LL * (long long)c->h_sc->host_writes;
  return SWF_OK;
}

int swf_set_host_mirror(swf_ctx* c, int on) {
  if (!c) return SWF_ECONFIG;
  c->host_mirror = on ? 1 : 0;
  c->mirror_valid = 0;
  return SWF_OK;
}

int swf_host_changed(swf_ctx* c) {
  if (!c) return SWF_ECONFIG;
  c->mirror_valid = 0;
  return SWF_OK;
}

int swf_debug_redo_counts(const swf_ctx* c, int* counts) {
  if (!c || !counts) return SWF_ECONFIG;
  counts[0] = c->h_sc->redo_n[0];
  counts[1] = c->h_sc->redo_n[1] + c->h_sc->redo_n[2];
  return SWF_OK;
}

int swf_debug_region_loads(const swf_ctx* c) {
  if (!c) return SWF_ECONFIG;
  return c->tma_ok ? 1 : 0;
}

int swf_last_ingest_bytes(const swf_ctx* c, long long* bytes) {
  if (!c || !bytes) return SWF_ECONFIG;
  *bytes = c->last_ingest_bytes;
  return SWF_OK;
}

int swf_run(swf_ctx* c, int n, double dt_cap, int* done, swf_step_info* last) {
  NvtxRange nv("swf_run");
  c->mirror_valid = 0;
  if (c->state_partial)
    return set_err(c, SWF_ECONFIG,
                   "the device state is incomplete after a pinned host-buffer step (sparse "
                   "momentum ingest); upload a state first");
  cudaSetDevice(c->device);
  if (done) *done = 0;
  if (n <= 0) return SWF_OK;
  c->last_staged = c->mode == 1;
  if (c->mode == 1) {
    for (int k = 0; k < n; ++k) {
      swf_step_info tmp;
      int rc = swf_step(c, dt_cap, last ? last : &tmp);
      if (rc) return rc;
      if (done) *done = k + 1;
    }
    return SWF_OK;
  }
  int cur0 = c->cur;
  int rc = reset_counters(c);
  if (rc) return rc;
  int enq = 0;
  // leading single step to reach an even buffer parity for the graph
  if (c->cur != 0) {
    if ((rc = fused_enqueue_step(c, dt_cap))) return rc;
    ++enq;
  }
  int pairs = (n - enq) / 2;
  if (pairs > 0) {
    if (c->timing) {
      for (int p = 0; p < 2 * pairs; ++p)
        if ((rc = fused_enqueue_step(c, dt_cap))) return rc;
    } else if (!c->graph || c->graph_dt_cap != dt_cap) {
      drop_graph(c);
      cudaGraph_t g;
      cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return cuda_check(c, e, "graph capture");
      bool saved = c->timing;
      c->timing = false;
      int rc1 = fused_enqueue_step(c, dt_cap);
      int rc2 = rc1 ? rc1 : fused_enqueue_step(c, dt_cap);
      c->timing = saved;
      e = cudaStreamEndCapture(c->stream, &g);
      if (rc2) return rc2;
      if (e != cudaSuccess) return cuda_check(c, e, "graph capture end");
      e = cudaGraphInstantiate(&c->graph, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_check(c, e, "graph instantiate");
      c->graph_dt_cap = dt_cap;
    }
    for (int p = 0; p < pairs && c->graph; ++p) {
      cudaError_t e = cudaGraphLaunch(c->graph, c->stream);
      if (e != cudaSuccess) return cuda_check(c, e, "graph launch");
    }
    enq += 2 * pairs;
    c->cur = 0;  // the captured pairs end on buffer 0
  }
  if (enq < n) {
    if ((rc = fused_enqueue_step(c, dt_cap))) return rc;
    ++enq;
  }
  if (last && (rc = fused_exact_volumes(c))) return rc;  // the last step's volumes
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "run");
  rc = commit_batch(c, cur0, enq, done);
  if (last && c->h_sc->steps_done > 0) fill_fused_info(c, last);
  return rc;
}

int swf_active_tiles(swf_ctx* c, int* n_active, int* n_total, int* cells_per_tile) {
  cudaSetDevice(c->device);
  size_t nt = (size_t)c->geo.tiles_x * c->geo.tiles_y;
  std::vector<unsigned char> f(nt ? nt : 1);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && nt)
    e = cudaMemcpy(f.data(), tile_act_at(c, 1 - c->cur), nt, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_check(c, e, "active tiles");
  int n = 0;
  for (size_t t = 0; t < nt; ++t) n += (f[t] & 2) ? 1 : 0;
  if (n_active) *n_active = n;
  if (n_total) *n_total = (int)nt;
  if (cells_per_tile) *cells_per_tile = 32 * 16;
  return SWF_OK;
}

int swf_sync(swf_ctx* c) {
  cudaSetDevice(c->device);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "sync");
  return check_device_error(c);
}

int swf_set_timing(swf_ctx* c, int slots) {
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (cudaEvent_t e : c->tev) cudaEventDestroy(e);
  c->tev.clear();
  c->tslots = 0;
  c->tstep = 0;
  c->timing = slots != 0;
  if (slots > 1) {
    c->tev.resize((size_t)slots * 6);
    for (auto& e : c->tev) {
      cudaError_t r = cudaEventCreate(&e);
      if (r != cudaSuccess) return cuda_check(c, r, "timing events");
    }
    c->tslots = slots;
  }
  drop_graph(c);
  return SWF_OK;
}

int swf_timing_read(swf_ctx* c, int nsteps, double* out) {
  cudaSetDevice(c->device);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "timing read");
  if (c->tslots <= 0) return set_err(c, SWF_ECONFIG, "per-step timing needs swf_set_timing(ctx, slots > 1)");
  if (nsteps > c->tslots || nsteps > c->tstep)
    return set_err(c, SWF_ECONFIG, "fewer timed steps recorded than requested");
  int map[5][2] = {{0, 0}, {1, 1}, {2, 2}, {3, 6}, {4, 7}};
  for (int s = 0; s < nsteps; ++s) {
    long long st = c->tstep - nsteps + s;
    const cudaEvent_t* E = &c->tev[(size_t)(st % c->tslots) * 6];
    double* o = out + (size_t)s * 8;
    for (int q = 0; q < 8; ++q) o[q] = 0.0;
    for (auto& m : map) {
      float ms = 0.f;
      e = cudaEventElapsedTime(&ms, E[m[0]], E[m[0] + 1]);
      if (e != cudaSuccess) return cuda_check(c, e, "timing elapsed");
      o[m[1]] = ms * 1e-3;
    }
  }
  return SWF_OK;
}

void* swf_stream(swf_ctx* c) { return (void*)c->stream; }

int swf_set_mode(swf_ctx* c, int mode) {
  if (mode != 0 && mode != 1) return set_err(c, SWF_ECONFIG, "mode must be 0 (fused) or 1 (staged)");
  c->mode = mode;
  return SWF_OK;
}

int swf_stage(swf_ctx* c, int stage, double arg, double* tau_out) {
  c->mirror_valid = 0;
  if (c->state_partial)
    return set_err(c, SWF_ECONFIG,
                   "the device state is incomplete after a pinned host-buffer step (sparse "
                   "momentum ingest); upload a state first");
  cudaSetDevice(c->device);
  if (stage == SWF_STAGE_BEGIN) {
    int rc = reset_counters(c);
    if (rc) return rc;
  }
  c->last_staged = 1;
  int rc = stage_run(c, stage, arg, tau_out);
  if (rc) return rc;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "stage");
  return SWF_OK;
}

int swf_download_scratch(swf_ctx* c, int which, double* out) {
  cudaSetDevice(c->device);
  return stage_download(c, which, out);
}

int swf_download_mask(swf_ctx* c, int* interior, int* halo, int* nbx, int* nby) {
  cudaSetDevice(c->device);
  const Geo& G = c->geo;
  size_t nb = (size_t)G.nbx * (G.bj1 - G.bj0);
  if (nbx) *nbx = G.nbx;
  if (nby) *nby = G.bj1 - G.bj0;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && interior && nb)
    e = cudaMemcpy(interior, c->d_interior, nb * sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && halo && nb) e = cudaMemcpy(halo, c->d_halo, nb * sizeof(int), cudaMemcpyDeviceToHost);
  return cuda_check(c, e, "download_mask");
}

int swf_last_volumes(swf_ctx* c, double* cd, double* sv, double* bo) {
  cudaSetDevice(c->device);
  double v[3] = {0, 0, 0};
  if (c->last_staged) {
    int rc = stage_volumes(c, v);
    if (rc) return rc;
  } else {
    cudaError_t e = cudaMemcpy(c->h_sc, c->d_sc, sizeof(StepScalars), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_check(c, e, "volumes");
    v[0] = c->h_sc->deficit;
    v[1] = c->h_sc->srcvol;
    v[2] = c->h_sc->outflow;
  }
  if (cd) *cd = v[0];
  if (sv) *sv = v[1];
  if (bo) *bo = v[2];
  return SWF_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// device-side KAT helpers (free functions evaluated on the GPU)
// ---------------------------------------------------------------------------
namespace {

__global__ void k_hll(int n, const double* in, double g, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* a = in + 6 * (size_t)i;
  FaceFlux f = hll_face_flux(a[0], a[1], a[2], a[3], a[4], a[5], g);
  out[3 * (size_t)i] = f.fm;
  out[3 * (size_t)i + 1] = f.fn;
  out[3 * (size_t)i + 2] = f.ft;
}

// out[2i] = rdiv(a, recip_of(b)) (shared-reciprocal division), out[2i+1] = a/b
__global__ void k_rdiv(int n, const double* in, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = in[2 * (size_t)i], b = in[2 * (size_t)i + 1];
  out[2 * (size_t)i] = rdiv(a, recip_of(b));
  out[2 * (size_t)i + 1] = a / b;
}

// speculative mode: out[2i] = fast-path quotient, out[2i+1] = 1.0 if accepted
__global__ void k_rdiv_spec(int n, const double* in, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = in[2 * (size_t)i], b = in[2 * (size_t)i + 1];
  bool ok = true;
  out[2 * (size_t)i] = rdiv(a, recip_of(b), &ok);
  out[2 * (size_t)i + 1] = ok ? 1.0 : 0.0;
}

// speculative square root: out[2i] = ssqrt(x, &ok), out[2i+1] = accepted,
// checked against the IEEE sqrt by the test
__global__ void k_sqrt_spec(int n, const double* x, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool ok = true;
  out[2 * (size_t)i] = ssqrt(x[i], &ok);
  out[2 * (size_t)i + 1] = ok ? 1.0 : 0.0;
}

__global__ void k_cbrt(int n, const double* x, double* y) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = glibc_cbrt(x[i]);
}

__global__ void k_fric(int n, const double* in, double g, double nm, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double fx, fy;
  friction_core(in[3 * (size_t)i], in[3 * (size_t)i + 1], in[3 * (size_t)i + 2], g, nm, fx, fy);
  out[2 * (size_t)i] = fx;
  out[2 * (size_t)i + 1] = fy;
}

template <class L>
int run_kat(size_t nin, const double* in, size_t nout, double* out, L&& launch) {
  double *din = nullptr, *dout = nullptr;
  cudaError_t e = cudaMalloc(&din, (nin ? nin : 1) * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&dout, (nout ? nout : 1) * sizeof(double));
  if (e == cudaSuccess && nin) e = cudaMemcpy(din, in, nin * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    launch(din, dout);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && nout) e = cudaMemcpy(out, dout, nout * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(din);
  cudaFree(dout);
  return cuda_check(nullptr, e, "device KAT");
}

}  // namespace

extern "C" {

int swf_dev_hll_face_flux(int n, const double* in, double g, double* out) {
  return run_kat(6 * (size_t)n, in, 3 * (size_t)n, out, [&](double* di, double* dout) {
    k_hll<<<(n + 255) / 256, 256>>>(n, di, g, dout);
  });
}

int swf_dev_rdiv(int n, const double* ab, double* out) {
  return run_kat(2 * (size_t)n, ab, 2 * (size_t)n, out, [&](double* di, double* dout) {
    k_rdiv<<<(n + 255) / 256, 256>>>(n, di, dout);
  });
}

int swf_dev_rdiv_spec(int n, const double* ab, double* out) {
  return run_kat(2 * (size_t)n, ab, 2 * (size_t)n, out, [&](double* di, double* dout) {
    k_rdiv_spec<<<(n + 255) / 256, 256>>>(n, di, dout);
  });
}

int swf_dev_sqrt_spec(int n, const double* x, double* out) {
  return run_kat((size_t)n, x, 2 * (size_t)n, out, [&](double* di, double* dout) {
    k_sqrt_spec<<<(n + 255) / 256, 256>>>(n, di, dout);
  });
}

int swf_dev_cbrt(int n, const double* x, double* y) {
  return run_kat((size_t)n, x, (size_t)n, y, [&](double* di, double* dout) {
    k_cbrt<<<(n + 255) / 256, 256>>>(n, di, dout);
  });
}

int swf_dev_bottom_friction(int n, const double* in, double g, double nm, double* out) {
  return run_kat(3 * (size_t)n, in, 2 * (size_t)n, out, [&](double* di, double* dout) {
    k_fric<<<(n + 255) / 256, 256>>>(n, di, g, nm, dout);
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// row strips (multi-GPU decomposition)
// ---------------------------------------------------------------------------
extern "C" {

// The forces of a strip step and its CFL speed; `part` as fused_enqueue_phase1
// (-1: with k_begin, -2: the caller has enqueued k_begin and the mask).
static int strip_phase1_body(swf_ctx* c, double dt_cap, double* speed_out, int part) {
  int rc = fused_enqueue_phase1(c, dt_cap, part);
  if (rc) return rc;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "strip phase 1");
  rc = check_device_error(c);
  if (rc) return rc;
  // the strip's CFL speed: max over the per-CTA slots (k_tau folds them
  // on the device in the single-context path)
  unsigned long long mb = c->h_sc->speed_bits;
  for (int q = 0; q < SPEED_SLOTS; ++q) mb = c->h_sc->speed_slots[q] > mb ? c->h_sc->speed_slots[q] : mb;
  if (speed_out) *speed_out = bitsd(mb);
  return SWF_OK;
}

int swf_strip_phase1(swf_ctx* c, double dt_cap, double* speed_out) {
  if (c->state_partial)
    return set_err(c, SWF_ECONFIG,
                   "the device state is incomplete after a pinned host-buffer step (sparse "
                   "momentum ingest); upload a state first");
  cudaSetDevice(c->device);
  int rc = reset_counters(c);
  if (rc) return rc;
  return strip_phase1_body(c, dt_cap, speed_out, -1);
}

int swf_strip_phase2(swf_ctx* c, double global_speed, double dt_cap, swf_step_info* info) {
  cudaSetDevice(c->device);
  int cur0 = c->cur;
  int rc = fused_enqueue_phase2(c, dt_cap, global_speed < 0.0 ? 0.0 : global_speed);
  if (rc) {
    c->cur = cur0;
    return rc;
  }
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "strip phase 2");
  rc = commit_batch(c, cur0, 1, nullptr);
  if (rc) return rc;
  if (info) fill_fused_info(c, info);
  return SWF_OK;
}

// ---- host-buffer step of a strip (pinned window arrays) ----------------------
static bool host_mapped(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer == p;
}

int swf_strip_host_phase1(swf_ctx* c, double* H, double* HUx, double* HUy, const double* t,
                          double dt_cap, double* speed_out) {
  cudaSetDevice(c->device);
  if (c->mode != 0) return set_err(c, SWF_ECONFIG, "strip host step needs the fused path");
  if (!host_mapped(H) || !host_mapped(HUx) || !host_mapped(HUy))
    return set_err(c, SWF_ECONFIG, "strip host step needs pinned (device-mapped) window arrays");
  const Geo& G = c->geo;
  int rc = reset_counters(c);
  if (rc) return rc;
  size_t n = local_cells(c), bytes = n * sizeof(double);
  cudaError_t e = cudaMemcpyAsync(c->H[c->cur], H, bytes, cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&c->d_sc->t, t, sizeof(double), cudaMemcpyHostToDevice, c->stream);
  // the ghost rows' momentum in full (their tiles belong to the neighbours)
  size_t nx = (size_t)G.nx, lo = (size_t)G.r0 * nx, hi0 = (size_t)G.r1 * nx;
  for (int f = 0; f < 2 && e == cudaSuccess; ++f) {
    double* dev = f == 0 ? c->HUx[c->cur] : c->HUy[c->cur];
    const double* host = f == 0 ? HUx : HUy;
    if (lo) e = cudaMemcpyAsync(dev, host, lo * sizeof(double), cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess && n > hi0)
      e = cudaMemcpyAsync(dev + hi0, host + hi0, (n - hi0) * sizeof(double), cudaMemcpyHostToDevice,
                          c->stream);
  }
  size_t nt = (size_t)G.tiles_x * G.tiles_y;
  if (e == cudaSuccess && nt) e = cudaMemsetAsync(c->d_tile_same, 0, nt, c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "strip host ingest");
  invalidate_mask(c);
  if ((rc = launch_begin(c, dt_cap)) || (rc = launch_mask(c)) || (rc = fused_ingest_hu(c, HUx, HUy)))
    return rc;
  // the owned tiles' flags describe this state: the forces list skips the
  // dry ones (ghost and edge tile rows are always visited)
  e = cudaMemsetAsync(&c->d_sc->mask_fresh, 1, sizeof(int), c->stream);
  if (e != cudaSuccess) return cuda_check(c, e, "strip host mask");
  c->state_partial = 0;
  c->last_ingest_bytes = (long long)bytes + 16LL * (long long)(lo + (n - hi0));
  // counters reset and k_begin / k_mask enqueued above: the forces only
  return strip_phase1_body(c, dt_cap, speed_out, -2);
}

int swf_strip_host_phase2(swf_ctx* c, double* H, double* HUx, double* HUy, double* t,
                          double global_speed, double dt_cap, swf_step_info* info) {
  cudaSetDevice(c->device);
  c->wt_host[0] = H;
  c->wt_host[1] = HUx;
  c->wt_host[2] = HUy;
  int rc = swf_strip_phase2(c, global_speed, dt_cap, info);
  c->wt_host[0] = c->wt_host[1] = c->wt_host[2] = nullptr;
  c->state_partial = 1;
  if (rc) {
    if (rc == SWF_ENUMERICAL && !fused_restore_host(c, H, HUx, HUy)) cudaStreamSynchronize(c->stream);
    return rc;
  }
  int na = 0, ntot = 0, cpt = 0;
  swf_active_tiles(c, &na, &ntot, &cpt);
  c->last_ingest_bytes += 2LL * 8 * na * cpt;
  if (t) *t = c->h_t;
  return SWF_OK;
}

int swf_strip_halo_ptrs(swf_ctx* c, int side, double** send3, double** recv3, size_t* count) {
  const Geo& G = c->geo;
  int ghosts = side == 0 ? G.r0 : G.rows - G.r1;
  size_t nx = G.nx;
  *count = (size_t)ghosts * nx;
  int rs = side == 0 ? G.r0 : G.r1 - ghosts;  // first owned row to send
  int rr = side == 0 ? 0 : G.r1;              // first ghost row to receive
  double* f[3] = {c->H[c->cur], c->HUx[c->cur], c->HUy[c->cur]};
  for (int q = 0; q < 3; ++q) {
    send3[q] = f[q] + (size_t)rs * nx;
    recv3[q] = f[q] + (size_t)rr * nx;
  }
  return SWF_OK;
}

// Pack the SWF_HALO owned boundary rows of (H, HUx, HUy) on `side` into a
// contiguous device buffer [H rows | HUx rows | HUy rows], or unpack a
// neighbour's pack into the ghost rows.  Enqueued on the context stream and
// synchronised, so the buffer can go straight to NCCL on another stream.
int swf_strip_pack(swf_ctx* c, int side, double* dst) {
  cudaSetDevice(c->device);
  double *s3[3], *r3[3];
  size_t count = 0;
  swf_strip_halo_ptrs(c, side, s3, r3, &count);
  cudaError_t e = cudaSuccess;
  for (int q = 0; q < 3 && e == cudaSuccess && count; ++q)
    e = cudaMemcpyAsync(dst + q * count, s3[q], count * sizeof(double), cudaMemcpyDeviceToDevice,
                        c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return cuda_check(c, e, "strip pack");
}

int swf_strip_unpack(swf_ctx* c, int side, const double* src) {
  cudaSetDevice(c->device);
  double *s3[3], *r3[3];
  size_t count = 0;
  swf_strip_halo_ptrs(c, side, s3, r3, &count);
  cudaError_t e = cudaSuccess;
  for (int q = 0; q < 3 && e == cudaSuccess && count; ++q)
    e = cudaMemcpyAsync(r3[q], src + q * count, count * sizeof(double), cudaMemcpyDeviceToDevice,
                        c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return cuda_check(c, e, "strip unpack");
}

// ---- asynchronous strip steps: no host round trip inside a batch ----------
int swf_strip_begin_batch(swf_ctx* c) {
  if (c->state_partial)
    return set_err(c, SWF_ECONFIG,
                   "the device state is incomplete after a pinned host-buffer step (sparse "
                   "momentum ingest); upload a state first");
  cudaSetDevice(c->device);
  if (c->mode != 0) return set_err(c, SWF_ECONFIG, "asynchronous strip steps need the fused path");
  int rc = reset_counters(c);
  if (rc) return rc;
  c->batch_cur0 = c->cur;
  c->batch_steps = 0;
  return SWF_OK;
}

int swf_strip_forces(swf_ctx* c, double dt_cap, int part) {
  cudaSetDevice(c->device);
  if (c->batch_cur0 < 0) return set_err(c, SWF_ECONFIG, "strip_forces outside a batch");
  if (part != 0 && part != 1) return set_err(c, SWF_ECONFIG, "strip_forces: part must be 0 or 1");
  return fused_enqueue_phase1(c, dt_cap, part);
}

int swf_strip_local_speed(swf_ctx* c, double* dev_out) {
  cudaSetDevice(c->device);
  return fused_local_speed(c, dev_out);
}

int swf_strip_finish(swf_ctx* c, const double* dev_global_speed, double dt_cap) {
  cudaSetDevice(c->device);
  if (c->batch_cur0 < 0) return set_err(c, SWF_ECONFIG, "strip_finish outside a batch");
  int rc = fused_enqueue_phase2(c, dt_cap, -1.0, dev_global_speed);
  if (rc) return rc;
  ++c->batch_steps;
  return SWF_OK;
}

int swf_strip_end_batch(swf_ctx* c, int* done, swf_step_info* last) {
  cudaSetDevice(c->device);
  if (c->batch_cur0 < 0) return set_err(c, SWF_ECONFIG, "strip_end_batch without a batch");
  cudaError_t e = cudaStreamSynchronize(c->stream);
  int cur0 = c->batch_cur0;
  c->batch_cur0 = -1;
  if (e != cudaSuccess) return cuda_check(c, e, "strip batch");
  int rc = commit_batch(c, cur0, c->batch_steps, done);
  if (last && c->h_sc->steps_done > 0) fill_fused_info(c, last);
  return rc;
}

int swf_strip_steps_done(const swf_ctx* c) { return c && c->h_sc ? c->h_sc->steps_done : 0; }

int swf_strip_settle(swf_ctx* c, int ok) {
  cudaSetDevice(c->device);
  const int done = c->h_sc->steps_done;
  if (ok == done) return SWF_OK;
  if (ok != done - 1 || ok < 0)
    return set_err(c, SWF_ECONFIG, "strip_settle: the strips are more than one step apart");
  // the step this strip finished beyond the others: its input buffer still
  // holds the state after `ok` steps (every strip stopped before the next
  // K4..K8), and k_finish kept the time before it
  cudaError_t e = cudaMemcpy(c->h_sc, c->d_sc, sizeof(StepScalars), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_check(c, e, "strip settle");
  const double t = c->h_sc->t_prev;
  c->h_sc->t = t;
  c->h_sc->steps_done = ok;
  e = cudaMemcpy(&c->d_sc->t, &t, sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(&c->d_sc->steps_done, &ok, sizeof(int), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_check(c, e, "strip settle");
  c->cur ^= 1;
  c->h_t = t;
  invalidate_mask(c);
  return SWF_OK;
}

int swf_strip_pack_async(swf_ctx* c, int side, double* dst) {
  cudaSetDevice(c->device);
  double *s3[3], *r3[3];
  size_t count = 0;
  swf_strip_halo_ptrs(c, side, s3, r3, &count);
  cudaError_t e = cudaSuccess;
  for (int q = 0; q < 3 && e == cudaSuccess && count; ++q)
    e = cudaMemcpyAsync(dst + q * count, s3[q], count * sizeof(double), cudaMemcpyDeviceToDevice,
                        c->stream);
  return cuda_check(c, e, "strip pack");
}

int swf_strip_unpack_async(swf_ctx* c, int side, const double* src) {
  cudaSetDevice(c->device);
  double *s3[3], *r3[3];
  size_t count = 0;
  swf_strip_halo_ptrs(c, side, s3, r3, &count);
  cudaError_t e = cudaSuccess;
  for (int q = 0; q < 3 && e == cudaSuccess && count; ++q)
    e = cudaMemcpyAsync(r3[q], src + q * count, count * sizeof(double), cudaMemcpyDeviceToDevice,
                        c->stream);
  // The ghost rows changed outside the fused path.  Their tiles' dry-skip
  // flags need no update: k_flist always lists a strip's ghost tile rows and
  // the tile rows next to its edges (the `edge` rule there), so no tile that
  // reads a ghost row is ever skipped on stale flags.
  return cuda_check(c, e, "strip unpack");
}

int swf_device_buffers(swf_ctx* c, double** out6) {
  if (!c || !out6) return SWF_ECONFIG;
  double* b[6] = {c->H[0], c->H[1], c->HUx[0], c->HUx[1], c->HUy[0], c->HUy[1]};
  for (int q = 0; q < 6; ++q) out6[q] = b[q];
  return SWF_OK;
}

int swf_strip_set_peer(swf_ctx* c, int side, double* const* bufs6, int peer_row0) {
  if (!c || side < 0 || side > 1) return SWF_ECONFIG;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (!bufs6) {
    c->peer_on[side] = 0;
  } else {
    const Geo& G = c->geo;
    bool has_ghosts = side == 0 ? G.r0 > 0 : G.r1 < G.rows;
    if (!has_ghosts) return set_err(c, SWF_ECONFIG, "strip_set_peer: no neighbour on that side");
    for (int f = 0; f < 3; ++f)
      for (int p = 0; p < 2; ++p) c->peer[side][f][p] = bufs6[2 * f + p];
    c->peer_drow[side] = G.jg0 - peer_row0;  // neighbour local row = ours + drow
    c->peer_on[side] = 1;
  }
  drop_graph(c);
  return SWF_OK;
}

int swf_strip_rows(const swf_ctx* c, int* j0, int* j1, int* glo, int* ghi) {
  const Geo& G = c->geo;
  if (j0) *j0 = G.jg0 + G.r0;
  if (j1) *j1 = G.jg0 + G.r1;
  if (glo) *glo = G.r0;
  if (ghi) *ghi = G.rows - G.r1;
  return SWF_OK;
}

int swf_device_count(int* n) {
  int k = 0;
  cudaError_t e = cudaGetDeviceCount(&k);
  if (n) *n = e == cudaSuccess ? k : 0;
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(nullptr, SWF_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  return SWF_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// single-process multi-GPU group (StepperOptions::devices > 1)
// ---------------------------------------------------------------------------
struct swf_group {
  std::vector<swf_ctx*> s;        // strips, ascending rows
  std::vector<double*> speed;     // per strip (its device): local CFL speed
  std::vector<double*> gspeed;    // per strip (its device): the group maximum
  double** d_in = nullptr;        // on strip 0's device: speed[] / gspeed[] pointers
  double** d_out = nullptr;
  StepScalars** d_sc = nullptr;   // on strip 0's device: every strip's step scalars
  std::vector<cudaEvent_t> ev_speed, ev_step;
  cudaEvent_t ev_max = nullptr;
  std::string err;
};

namespace {

// the exact maximum of the strips' speeds (non-negative doubles), written to
// every strip's device (peer stores).  It also stops the whole group once any
// strip has aborted: a per-cell error (CFL displacement, non-finite flux) in
// one strip's k_step of step k is seen here in step k+1 (this kernel runs
// after every strip's phase 1 of k+1, hence after every k_step of k), and the
// other strips get ERR_PEER, so none of them runs k_step of k+1.  Every strip
// then holds its committed state of step k in the parity buffer the commit
// picks (swf_group_run), and no healthy strip has overwritten it.
__global__ void k_group_max(double* const* in, double* const* out, StepScalars* const* sc,
                            int n) {
  if (threadIdx.x != 0) return;
  bool stop = false;
  for (int d = 0; d < n; ++d) stop = stop || *(volatile unsigned long long*)&sc[d]->err_key != ERR_NONE;
  if (stop) {
    for (int d = 0; d < n; ++d) atomicMin(&sc[d]->err_key, ERR_PEER << 58);
    return;
  }
  double m = 0.0;
  for (int d = 0; d < n; ++d) m = in[d][0] > m ? in[d][0] : m;
  for (int d = 0; d < n; ++d) out[d][0] = m;
}

int group_err(swf_group* g, int rc, const std::string& m) {
  g->err = m;
  g_err = m;
  return rc;
}

int enable_peer(int a, int b) {
  if (a == b) return SWF_OK;
  int can = 0;
  cudaDeviceCanAccessPeer(&can, a, b);
  if (!can) return SWF_ECUDA;
  cudaSetDevice(a);
  cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  return e == cudaSuccess ? SWF_OK : SWF_ECUDA;
}

}  // namespace

extern "C" {

void swf_group_destroy(swf_group* g) {
  if (!g) return;
  for (size_t d = 0; d < g->s.size(); ++d) {
    cudaSetDevice(g->s[d]->device);
    cudaStreamSynchronize(g->s[d]->stream);
    for (int side = 0; side < 2; ++side) swf_strip_set_peer(g->s[d], side, nullptr, 0);
    if (d < g->speed.size()) cudaFree(g->speed[d]);
    if (d < g->gspeed.size()) cudaFree(g->gspeed[d]);
    if (d < g->ev_speed.size()) cudaEventDestroy(g->ev_speed[d]);
    if (d < g->ev_step.size()) cudaEventDestroy(g->ev_step[d]);
  }
  if (!g->s.empty()) {
    cudaSetDevice(g->s[0]->device);
    cudaFree(g->d_in);
    cudaFree(g->d_out);
    cudaFree(g->d_sc);
    if (g->ev_max) cudaEventDestroy(g->ev_max);
  }
  delete g;
}

int swf_group_create(swf_ctx* const* strips, int n, swf_group** out) {
  if (!out || !strips || n < 1) return set_err(nullptr, SWF_ECONFIG, "group: no strips");
  *out = nullptr;
  for (int d = 0; d < n; ++d) {
    if (!strips[d]) return set_err(nullptr, SWF_ECONFIG, "group: null strip");
    const Geo& G = strips[d]->geo;
    if (d > 0) {
      const Geo& P = strips[d - 1]->geo;
      if (P.jg0 + P.r1 != G.jg0 + G.r0 || P.nx != G.nx || P.ny != G.ny)
        return set_err(nullptr, SWF_ECONFIG, "group: strips must be adjacent rows of one grid");
    }
    if (strips[d]->mode != 0) return set_err(nullptr, SWF_ECONFIG, "group: strips need the fused path");
  }
  swf_group* g = new swf_group();
  g->s.assign(strips, strips + n);
  const int dev0 = strips[0]->device;
  // peer access: every device with the first (the speed reduction) and with
  // its neighbours (the halo stores)
  for (int d = 0; d < n; ++d) {
    int a = strips[d]->device;
    int rc = enable_peer(dev0, a) | enable_peer(a, dev0);
    if (d > 0) rc |= enable_peer(a, strips[d - 1]->device) | enable_peer(strips[d - 1]->device, a);
    if (rc) {
      swf_group_destroy(g);
      return set_err(nullptr, SWF_ECUDA, "group: peer access between the devices is unavailable");
    }
  }
  cudaError_t e = cudaSuccess;
  g->speed.assign(n, nullptr);
  g->gspeed.assign(n, nullptr);
  g->ev_speed.assign(n, nullptr);
  g->ev_step.assign(n, nullptr);
  for (int d = 0; d < n && e == cudaSuccess; ++d) {
    cudaSetDevice(strips[d]->device);
    e = cudaMalloc(&g->speed[d], sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&g->gspeed[d], sizeof(double));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_speed[d], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_step[d], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) {
    cudaSetDevice(dev0);
    e = cudaMalloc(&g->d_in, n * sizeof(double*));
    if (e == cudaSuccess) e = cudaMalloc(&g->d_out, n * sizeof(double*));
    if (e == cudaSuccess) e = cudaMemcpy(g->d_in, g->speed.data(), n * sizeof(double*), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_out, g->gspeed.data(), n * sizeof(double*), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_sc, n * sizeof(StepScalars*));
    if (e == cudaSuccess) {
      std::vector<StepScalars*> scs(n);
      for (int d = 0; d < n; ++d) scs[d] = strips[d]->d_sc;
      e = cudaMemcpy(g->d_sc, scs.data(), n * sizeof(StepScalars*), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->ev_max, cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    std::string m = std::string("group setup: ") + cudaGetErrorString(e);
    swf_group_destroy(g);
    return set_err(nullptr, SWF_ECUDA, m);
  }
  // each k_step stores its boundary rows into the neighbours' ghost rows
  for (int d = 0; d < n; ++d) {
    for (int side = 0; side < 2; ++side) {
      int nb = side == 0 ? d - 1 : d + 1;
      if (nb < 0 || nb >= n) continue;
      double* bufs[6];
      swf_device_buffers(strips[nb], bufs);
      int rc = swf_strip_set_peer(strips[d], side, bufs, strips[nb]->geo.jg0);
      if (rc) {
        std::string m = strips[d]->err;
        swf_group_destroy(g);
        return set_err(nullptr, rc, m);
      }
    }
  }
  *out = g;
  return SWF_OK;
}

const char* swf_group_last_error(const swf_group* g) { return g ? g->err.c_str() : g_err.c_str(); }

int swf_group_run(swf_group* g, int nsteps, double dt_cap, int* done, swf_step_info* last) {
  if (!g) return set_err(nullptr, SWF_ECONFIG, "group: null");
  if (done) *done = 0;
  const int n = (int)g->s.size();
  std::vector<int> cur0(n);
  for (int d = 0; d < n; ++d) {
    swf_ctx* c = g->s[d];
    if (c->state_partial) return group_err(g, SWF_ECONFIG, "group: upload a state first");
    if (c->cur != g->s[0]->cur) return group_err(g, SWF_ECONFIG, "group: strips out of step");
    cudaSetDevice(c->device);
    int rc = reset_counters(c);
    if (rc) return group_err(g, rc, c->err);
    cur0[d] = c->cur;
  }
  int rc = SWF_OK;
  for (int k = 0; k < nsteps && !rc; ++k) {
    // interior tile rows first (no ghost row read), on every device
    for (int d = 0; d < n && !rc; ++d) {
      cudaSetDevice(g->s[d]->device);
      rc = fused_enqueue_phase1(g->s[d], dt_cap, 0);
    }
    // the ghost-dependent rows after the neighbours' previous k_step
    for (int d = 0; d < n && !rc; ++d) {
      swf_ctx* c = g->s[d];
      cudaSetDevice(c->device);
      if (k > 0)
        for (int nb = d - 1; nb <= d + 1; nb += 2)
          if (nb >= 0 && nb < n) cudaStreamWaitEvent(c->stream, g->ev_step[nb], 0);
      rc = fused_enqueue_phase1(c, dt_cap, 1);
      if (!rc) rc = fused_local_speed(c, g->speed[d]);
      if (!rc) cudaEventRecord(g->ev_speed[d], c->stream);
    }
    if (rc) break;
    swf_ctx* c0 = g->s[0];
    cudaSetDevice(c0->device);
    for (int d = 0; d < n; ++d) cudaStreamWaitEvent(c0->stream, g->ev_speed[d], 0);
    k_group_max<<<1, 32, 0, c0->stream>>>(g->d_in, g->d_out, g->d_sc, n);
    cudaEventRecord(g->ev_max, c0->stream);
    for (int d = 0; d < n && !rc; ++d) {
      swf_ctx* c = g->s[d];
      cudaSetDevice(c->device);
      cudaStreamWaitEvent(c->stream, g->ev_max, 0);
      rc = fused_enqueue_phase2(c, dt_cap, -1.0, g->gspeed[d]);
      if (!rc) cudaEventRecord(g->ev_step[d], c->stream);
    }
  }
  // every strip commits the steps all of them completed
  int ok = nsteps, first_rc = rc, first = -1;
  std::vector<int> rcs(n);
  for (int d = 0; d < n; ++d) {
    swf_ctx* c = g->s[d];
    cudaSetDevice(c->device);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    rcs[d] = e != cudaSuccess ? cuda_check(c, e, "group run") : check_device_error(c);
    // a strip stopped only because another one aborted reports nothing itself
    if (rcs[d] == SWF_ENUMERICAL && (c->h_sc->err_key >> 58) == ERR_PEER) rcs[d] = SWF_OK;
    ok = std::min(ok, c->h_sc->steps_done);
    if (rcs[d] && (first < 0 || (rcs[d] == SWF_ENUMERICAL && rcs[first] != SWF_ENUMERICAL))) first = d;
  }
  double t = 0.0;
  for (int d = 0; d < n; ++d)
    if (g->s[d]->h_sc->steps_done == ok) t = g->s[d]->h_sc->t;
  for (int d = 0; d < n; ++d) {
    swf_ctx* c = g->s[d];
    cudaSetDevice(c->device);
    if (c->h_sc->steps_done != ok) {  // discard the steps the others did not finish
      c->h_sc->t = t;
      cudaMemcpy(&c->d_sc->t, &t, sizeof(double), cudaMemcpyHostToDevice);
      invalidate_mask(c);
    }
    c->cur = (cur0[d] + ok) & 1;
    c->h_t = t;
  }
  if (done) *done = ok;
  if (last && ok > 0) {
    swf_step_info sum{};
    long long flux_act = 0;
    for (int d = 0; d < n; ++d) {
      flux_act += g->s[d]->h_sc->flux_act;
      swf_step_info a{};
      fill_fused_info(g->s[d], &a);
      if (d == 0) {
        sum = a;
      } else {
        sum.lagrangian_blocks += a.lagrangian_blocks;
        sum.flux_blocks += a.flux_blocks;
        sum.total_blocks += a.total_blocks;
        sum.clamp_deficit_volume += a.clamp_deficit_volume;
        sum.source_volume += a.source_volume;
        sum.boundary_outflow_volume += a.boundary_outflow_volume;
      }
    }
    sum.active_fraction = sum.total_blocks ? (double)flux_act / sum.total_blocks : 0.0;
    *last = sum;
  }
  if (first_rc) return group_err(g, first_rc, g->s[0]->err);
  if (first >= 0) return group_err(g, rcs[first], g->s[first]->err);
  return SWF_OK;
}

}  // extern "C"
