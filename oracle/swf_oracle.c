/*
 * swf_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C, single-threaded restatement of the CSPH-TVD time step of the
 * reference (arXiv 1705.00614 `swflood`, /root/reference/proj), written from
 * the reference's behaviour, not copied.  Every function cites the file:line
 * it restates.  Arithmetic follows the reference's operation order exactly
 * (parenthesised below) and is compiled with -ffp-contract=off, so that the
 * results are bit-identical to the reference built with its pinned flags
 * (oracle/Makefile) and to the CUDA PARITY path built with -fmad=false.
 *
 * Parity pin: tests/test_oracle_pin.py checks this file bit-for-bit against
 * the real reference (oracle/_ref/libswflood_ref.so, built by oracle/Makefile)
 * on every stage and scratch array, and against the committed golden vectors
 * in tests/golden/ (generated from the real reference by
 * tests/golden/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
 * load liborc.so; the product path never does.
 */
#include "swf_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* helpers mirroring std::min / std::max / minmod exactly                    */
/* ------------------------------------------------------------------------ */

/* std::min(a,b) == (b < a) ? b : a ; std::max(a,b) == (a < b) ? b : a */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }

/* stepper.cpp:23-27 */
static inline double minmod(double a, double b) {
  if (a > 0.0 && b > 0.0) return smin(a, b);
  if (a < 0.0 && b < 0.0) return smax(a, b);
  return 0.0;
}

/* glibc 2.39 sysdeps/ieee754/dbl-64/s_cbrt.c, the libm cbrt the reference
 * calls at forcing.hpp:81 and stepper.cpp:292,366.
 * It is third-party arithmetic, restated here so the parity contract does not
 * depend on the host libm; tests pin it against libm bit-for-bit. */
double orc_cbrt(double x) {
  static const double factor[5] = {1.0 / 1.5874010519681994748, 1.0 / 1.2599210498948731648,
                                   1.0, 1.2599210498948731648, 1.5874010519681994748};
  int xe;
  double xm = frexp(fabs(x), &xe);
  if (xe == 0 && (x == 0.0 || isnan(x) || isinf(x))) return x + x;
  double u = (0.354895765043919860 +
              ((1.50819193781584896 +
                ((-2.11499494167371287 +
                  ((2.44693122563534430 +
                    ((-1.83469277483613086 + (0.784932344976639262 - 0.145263899385486377 * xm) * xm) *
                     xm)) *
                   xm)) *
                 xm)) *
               xm));
  double t2 = u * u * u;
  double ym = u * (t2 + 2.0 * xm) / (2.0 * t2 + xm) * factor[2 + xe % 3];
  return ldexp(x > 0.0 ? ym : -ym, xe / 3);
}

/* ------------------------------------------------------------------------ */
/* context                                                                   */
/* ------------------------------------------------------------------------ */

typedef struct {
  int kind, i0, j0, i1, j1, nh;
  double *ht, *hq;
  double rate, vx, vy;
} src_spec;

typedef struct {
  double fm, fnl, fnr, ft;
} face_rec; /* FaceRec, stepper.hpp:124-129 */

struct orc_ctx {
  int nx, ny;
  double h, x0, y0;
  double* b;
  swf_params p; /* p.n_field points at nfield or NULL */
  double* nfield;
  swf_control ctl;
  swf_options opt;
  /* WindForcing (grid.hpp:87-95) */
  int nwind;
  double *wt, *wx, *wy;
  /* SourceSpec list (sources.hpp:25-36) */
  int nsrc;
  src_spec* src;
  /* FlowState */
  double *H, *HUx, *HUy, t;
  /* BlockMask (block.hpp:20-36) + dispatch lists (stepper.hpp:150) */
  int bs, nbx, nby;
  int *interior, *halo;
  int *lag, nlag, *flx, nflx, *skp, nskp;
  /* SourceField at t_n and sigma at t_mid (stepper.hpp:151-152) */
  double *sigma, *svx, *svy, *sigma_mid;
  uint8_t* q;
  /* ForceField f_n, f_mid (forcing.hpp:16-25) */
  double *fn_fx, *fn_fy, *fn_rx, *fn_ry, *fn_sig;
  double *fm_fx, *fm_fy, *fm_rx, *fm_ry, *fm_sig;
  /* stage scratch (stepper.hpp:155-159) */
  double *hH, *hHUx, *hHUy, *Ht, *HVtx, *HVty, *drx, *dry, *Fh, *Fvx, *Fvy;
  face_rec *xf, *yf;
  double *blk_reduce, *blk_srcvol;
  long long* blk_err;
  double clamp_deficit, source_volume, boundary_outflow;
  char err[512];
};

static char g_err[512];

static int fail(orc_ctx* c, int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(c ? c->err : g_err, 512, fmt, ap);
  va_end(ap);
  return code;
}

static double* dalloc(size_t n) { return (double*)calloc(n ? n : 1, sizeof(double)); }

static size_t cells(const orc_ctx* c) { return (size_t)c->nx * (size_t)c->ny; }

/* ------------------------------------------------------------------------ */
/* validation: grid.cpp:13-21, grid.cpp:42-51, stepper.cpp:31-37,136-139    */
/* ------------------------------------------------------------------------ */

static int validate_control(orc_ctx* c, const swf_control* k) {
  if (!(k->courant > 0.0 && k->courant < 1.0))
    return fail(c, SWF_ECONFIG, "timestep: Courant number must be in (0,1)");
  if (!(k->dt_max > 0.0)) return fail(c, SWF_ECONFIG, "timestep: dt_max must be positive");
  if (!(k->dt_min > 0.0 && k->dt_min < k->dt_max))
    return fail(c, SWF_ECONFIG, "timestep: need 0 < dt_min < dt_max");
  return SWF_OK;
}

static int validate_setup(const swf_terrain* T, const swf_params* P) {
  if (T->nx < 1 || T->ny < 1) return fail(NULL, SWF_ECONFIG, "terrain: nx and ny must be >= 1");
  if (!(T->h > 0.0)) return fail(NULL, SWF_ECONFIG, "terrain: cell size must be positive");
  if (!T->b) return fail(NULL, SWF_ECONFIG, "terrain: bed array size mismatch");
  size_t n = (size_t)T->nx * (size_t)T->ny;
  for (size_t k = 0; k < n; ++k)
    if (!isfinite(T->b[k]))
      return fail(NULL, SWF_ECONFIG, "terrain: non-finite bed elevation at cell %zu", k);
  if (!(P->g > 0.0)) return fail(NULL, SWF_ECONFIG, "params: gravity must be positive");
  if (P->n_manning < 0.0) return fail(NULL, SWF_ECONFIG, "params: Manning coefficient must be >= 0");
  if (P->n_field)
    for (size_t k = 0; k < n; ++k)
      if (P->n_field[k] < 0.0) return fail(NULL, SWF_ECONFIG, "params: Manning field must be >= 0");
  if (P->nu < 0.0) return fail(NULL, SWF_ECONFIG, "params: viscosity must be >= 0");
  if (!(P->rho_water > 0.0)) return fail(NULL, SWF_ECONFIG, "params: water density must be positive");
  if (P->rho_air < 0.0) return fail(NULL, SWF_ECONFIG, "params: air density must be >= 0");
  if (!(P->eps_dry > 0.0)) return fail(NULL, SWF_ECONFIG, "params: dry threshold must be positive");
  return SWF_OK;
}

/* ------------------------------------------------------------------------ */
/* lifecycle: stepper.cpp:127-159                                            */
/* ------------------------------------------------------------------------ */

static void free_masklists(orc_ctx* c) {
  free(c->interior); free(c->halo); free(c->lag); free(c->flx); free(c->skp);
  free(c->blk_reduce); free(c->blk_srcvol); free(c->blk_err);
  c->interior = c->halo = c->lag = c->flx = c->skp = NULL;
  c->blk_reduce = c->blk_srcvol = NULL;
  c->blk_err = NULL;
}

static void free_sources(orc_ctx* c) {
  for (int s = 0; s < c->nsrc; ++s) { free(c->src[s].ht); free(c->src[s].hq); }
  free(c->src);
  c->src = NULL;
  c->nsrc = 0;
}

void orc_destroy(orc_ctx* c) {
  if (!c) return;
  double* arrs[] = {c->b, c->nfield, c->wt, c->wx, c->wy, c->H, c->HUx, c->HUy,
                    c->sigma, c->svx, c->svy, c->sigma_mid, c->fn_fx, c->fn_fy, c->fn_rx,
                    c->fn_ry, c->fn_sig, c->fm_fx, c->fm_fy, c->fm_rx, c->fm_ry, c->fm_sig,
                    c->hH, c->hHUx, c->hHUy, c->Ht, c->HVtx, c->HVty, c->drx, c->dry,
                    c->Fh, c->Fvx, c->Fvy};
  for (size_t k = 0; k < sizeof arrs / sizeof arrs[0]; ++k) free(arrs[k]);
  free(c->q); free(c->xf); free(c->yf);
  free_masklists(c);
  free_sources(c);
  free(c);
}

int orc_create(const swf_terrain* T, const swf_params* P, const swf_control* K,
               const swf_options* O, orc_ctx** out) {
  *out = NULL;
  int rc = validate_setup(T, P);
  if (rc) return rc;
  orc_ctx* c = (orc_ctx*)calloc(1, sizeof *c);
  rc = validate_control(NULL, K);
  if (rc) { free(c); return rc; }
  if (O->block_size < 1) { free(c); return fail(NULL, SWF_ECONFIG, "stepper: block size must be >= 1"); }
  c->nx = T->nx; c->ny = T->ny; c->h = T->h; c->x0 = T->x0; c->y0 = T->y0;
  size_t n = cells(c);
  c->b = dalloc(n);
  memcpy(c->b, T->b, n * sizeof(double));
  c->p = *P;
  if (P->n_field) {
    c->nfield = dalloc(n);
    memcpy(c->nfield, P->n_field, n * sizeof(double));
    c->p.n_field = c->nfield;
  }
  c->ctl = *K;
  c->opt = *O;
  if (c->opt.workers < 1) c->opt.workers = 1;
  c->H = dalloc(n); c->HUx = dalloc(n); c->HUy = dalloc(n);
  c->sigma = dalloc(n); c->svx = dalloc(n); c->svy = dalloc(n); c->sigma_mid = dalloc(n);
  c->q = (uint8_t*)calloc(n, 1);
  c->fn_fx = dalloc(n); c->fn_fy = dalloc(n); c->fn_rx = dalloc(n); c->fn_ry = dalloc(n); c->fn_sig = dalloc(n);
  c->fm_fx = dalloc(n); c->fm_fy = dalloc(n); c->fm_rx = dalloc(n); c->fm_ry = dalloc(n); c->fm_sig = dalloc(n);
  c->hH = dalloc(n); c->hHUx = dalloc(n); c->hHUy = dalloc(n);
  c->Ht = dalloc(n); c->HVtx = dalloc(n); c->HVty = dalloc(n);
  c->drx = dalloc(n); c->dry = dalloc(n);
  c->Fh = dalloc(n); c->Fvx = dalloc(n); c->Fvy = dalloc(n);
  c->xf = (face_rec*)calloc((size_t)(c->nx + 1) * c->ny, sizeof(face_rec));
  c->yf = (face_rec*)calloc((size_t)c->nx * (c->ny + 1), sizeof(face_rec));
  *out = c;
  return SWF_OK;
}

const char* orc_last_error(const orc_ctx* c) { return c ? c->err : g_err; }

/* WindForcing::validate, grid.cpp:77-82 */
int orc_set_wind(orc_ctx* c, int n, const double* t, const double* wx, const double* wy) {
  for (int k = 1; k < n; ++k)
    if (!(t[k] > t[k - 1])) return fail(c, SWF_ECONFIG, "wind: sample times must be strictly increasing");
  free(c->wt); free(c->wx); free(c->wy);
  c->nwind = n;
  c->wt = dalloc(n); c->wx = dalloc(n); c->wy = dalloc(n);
  for (int k = 0; k < n; ++k) { c->wt[k] = t[k]; c->wx[k] = wx[k]; c->wy[k] = wy[k]; }
  return SWF_OK;
}

/* SourceSpec::validate, sources.cpp:22-33 */
static int validate_source(orc_ctx* c, const swf_source* s, int idx) {
  if (s->i0 > s->i1 || s->j0 > s->j1)
    return fail(c, SWF_ECONFIG, "source 'src%d': empty cell rectangle", idx);
  int in0 = s->i0 >= 0 && s->i0 < c->nx && s->j0 >= 0 && s->j0 < c->ny;
  int in1 = s->i1 >= 0 && s->i1 < c->nx && s->j1 >= 0 && s->j1 < c->ny;
  if (!in0 || !in1) return fail(c, SWF_ECONFIG, "source 'src%d': cells outside grid", idx);
  for (int m = 1; m < s->n_hydro; ++m)
    if (!(s->hydro_t[m] > s->hydro_t[m - 1]))
      return fail(c, SWF_ECONFIG, "source 'src%d': hydrograph times must be strictly increasing", idx);
  if (s->kind == SWF_SOURCE_DISCHARGE && s->n_hydro <= 0)
    return fail(c, SWF_ECONFIG, "source 'src%d': discharge source needs a hydrograph", idx);
  return SWF_OK;
}

/* set_sources, stepper.cpp:166-170 */
int orc_set_sources(orc_ctx* c, int n, const swf_source* s) {
  for (int k = 0; k < n; ++k) {
    int rc = validate_source(c, &s[k], k);
    if (rc) return rc;
  }
  free_sources(c);
  c->nsrc = n;
  c->src = (src_spec*)calloc((size_t)(n > 0 ? n : 1), sizeof(src_spec));
  for (int k = 0; k < n; ++k) {
    src_spec* d = &c->src[k];
    d->kind = s[k].kind; d->i0 = s[k].i0; d->j0 = s[k].j0; d->i1 = s[k].i1; d->j1 = s[k].j1;
    d->nh = s[k].n_hydro;
    d->ht = dalloc(d->nh); d->hq = dalloc(d->nh);
    for (int m = 0; m < d->nh; ++m) { d->ht[m] = s[k].hydro_t[m]; d->hq[m] = s[k].hydro_q[m]; }
    d->rate = s[k].rate; d->vx = s[k].vx; d->vy = s[k].vy;
  }
  if (n == 0) { /* src_.clear_values(), grid.cpp:94-99 */
    size_t N = cells(c);
    memset(c->sigma, 0, N * sizeof(double));
    memset(c->svx, 0, N * sizeof(double));
    memset(c->svy, 0, N * sizeof(double));
    memset(c->q, 0, N);
  }
  return SWF_OK;
}

int orc_set_control(orc_ctx* c, const swf_control* k) {
  /* control() is a plain mutable reference in the reference (stepper.hpp:100):
   * no validation on assignment. */
  c->ctl = *k;
  return SWF_OK;
}

int orc_set_options(orc_ctx* c, const swf_options* o) {
  c->opt = *o; /* options() is a plain mutable reference (stepper.hpp:101) */
  return SWF_OK;
}

int orc_set_state(orc_ctx* c, const double* H, const double* HUx, const double* HUy, double t) {
  size_t n = cells(c);
  memcpy(c->H, H, n * sizeof(double));
  memcpy(c->HUx, HUx, n * sizeof(double));
  memcpy(c->HUy, HUy, n * sizeof(double));
  c->t = t;
  return SWF_OK;
}

int orc_get_state(orc_ctx* c, double* H, double* HUx, double* HUy, double* t) {
  size_t n = cells(c);
  memcpy(H, c->H, n * sizeof(double));
  memcpy(HUx, c->HUx, n * sizeof(double));
  memcpy(HUy, c->HUy, n * sizeof(double));
  if (t) *t = c->t;
  return SWF_OK;
}

/* ------------------------------------------------------------------------ */
/* time series: WindForcing::at grid.cpp:64-75, discharge_at sources.cpp:10-20 */
/* ------------------------------------------------------------------------ */

/* first index m with t < ts[m] (std::upper_bound) */
static int upper(const double* ts, int n, double t) {
  int lo = 0, len = n;
  while (len > 0) {
    int half = len / 2;
    if (!(t < ts[lo + half])) { lo += half + 1; len -= half + 1; }
    else len = half;
  }
  return lo;
}

static void wind_at(const orc_ctx* c, double t, double* wx, double* wy) {
  int n = c->nwind;
  if (n == 0) { *wx = 0.0; *wy = 0.0; return; }
  if (n == 1 || t <= c->wt[0]) { *wx = c->wx[0]; *wy = c->wy[0]; return; }
  if (t >= c->wt[n - 1]) { *wx = c->wx[n - 1]; *wy = c->wy[n - 1]; return; }
  int hi = upper(c->wt, n, t), lo = hi - 1;
  double a = (t - c->wt[lo]) / (c->wt[hi] - c->wt[lo]);
  *wx = c->wx[lo] + a * (c->wx[hi] - c->wx[lo]);
  *wy = c->wy[lo] + a * (c->wy[hi] - c->wy[lo]);
}

static double discharge_at(const src_spec* s, double t) {
  int n = s->nh;
  if (n == 0) return 0.0;
  if (n == 1 || t <= s->ht[0]) return s->hq[0];
  if (t >= s->ht[n - 1]) return s->hq[n - 1];
  int hi = upper(s->ht, n, t), lo = hi - 1;
  double a = (t - s->ht[lo]) / (s->ht[hi] - s->ht[lo]);
  return s->hq[lo] + a * (s->hq[hi] - s->hq[lo]);
}

/* cell_sigma, sources.cpp:37-41 */
static double cell_sigma(const orc_ctx* c, const src_spec* s, double t) {
  if (s->kind == SWF_SOURCE_RAIN) return s->rate;
  double q = discharge_at(s, t);
  int count = (s->i1 - s->i0 + 1) * (s->j1 - s->j0 + 1);
  return q / ((double)count * (c->h * c->h));
}

/* source_terms, sources.cpp:45-64 (into the context's SourceField) */
static void source_terms(orc_ctx* c, double t) {
  size_t N = cells(c);
  memset(c->sigma, 0, N * sizeof(double));
  memset(c->svx, 0, N * sizeof(double));
  memset(c->svy, 0, N * sizeof(double));
  for (int s = 0; s < c->nsrc; ++s) {
    const src_spec* sp = &c->src[s];
    double sig = cell_sigma(c, sp, t);
    for (int j = sp->j0; j <= sp->j1; ++j)
      for (int i = sp->i0; i <= sp->i1; ++i) {
        size_t k = (size_t)i + (size_t)j * c->nx;
        c->sigma[k] += sig;
        c->svx[k] = sp->vx;
        c->svy[k] = sp->vy;
      }
  }
  for (size_t k = 0; k < N; ++k) c->q[k] = (c->sigma[k] != 0.0) ? 1 : 0;
}

/* resample_sigma, sources.cpp:66-75 */
static void resample_sigma(orc_ctx* c, double t, double* out) {
  memset(out, 0, cells(c) * sizeof(double));
  for (int s = 0; s < c->nsrc; ++s) {
    const src_spec* sp = &c->src[s];
    double sig = cell_sigma(c, sp, t);
    for (int j = sp->j0; j <= sp->j1; ++j)
      for (int i = sp->i0; i <= sp->i1; ++i) out[(size_t)i + (size_t)j * c->nx] += sig;
  }
}

/* ------------------------------------------------------------------------ */
/* K1 block mask: block.cpp:7-87, stepper.cpp:172-201                        */
/* ------------------------------------------------------------------------ */

static void block_rect(const orc_ctx* c, int ib, int* i0, int* j0, int* i1, int* j1) {
  int bi = ib % c->nbx, bj = ib / c->nbx;
  *i0 = bi * c->bs;
  *j0 = bj * c->bs;
  *i1 = *i0 + c->bs - 1; if (*i1 > c->nx - 1) *i1 = c->nx - 1;
  *j1 = *j0 + c->bs - 1; if (*j1 > c->ny - 1) *j1 = c->ny - 1;
}

static int cell_wet(const orc_ctx* c, int i, int j) {
  size_t k = (size_t)i + (size_t)j * c->nx;
  return c->H[k] > c->p.eps_dry || c->q[k] != 0;
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

static void compute_block_mask(orc_ctx* c) {
  c->bs = c->opt.block_size;
  c->nbx = (c->nx + c->bs - 1) / c->bs;
  c->nby = (c->ny + c->bs - 1) / c->bs;
  int nb = c->nbx * c->nby;
  free_masklists(c);
  c->interior = (int*)calloc(nb, sizeof(int));
  c->halo = (int*)calloc(nb, sizeof(int));
  for (int ib = 0; ib < nb; ++ib) {
    int i0, j0, i1, j1, in = 0, ring = 0;
    block_rect(c, ib, &i0, &j0, &i1, &j1);
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) in += cell_wet(c, i, j);
    /* one-cell ring including corners, positions clamped into the domain */
    for (int i = i0 - 1; i <= i1 + 1; ++i) {
      ring += cell_wet(c, clampi(i, 0, c->nx - 1), clampi(j0 - 1, 0, c->ny - 1));
      ring += cell_wet(c, clampi(i, 0, c->nx - 1), clampi(j1 + 1, 0, c->ny - 1));
    }
    for (int j = j0; j <= j1; ++j) {
      ring += cell_wet(c, clampi(i0 - 1, 0, c->nx - 1), clampi(j, 0, c->ny - 1));
      ring += cell_wet(c, clampi(i1 + 1, 0, c->nx - 1), clampi(j, 0, c->ny - 1));
    }
    c->interior[ib] = in;
    c->halo[ib] = ring;
  }
  c->lag = (int*)malloc(sizeof(int) * (size_t)(nb > 0 ? nb : 1));
  c->flx = (int*)malloc(sizeof(int) * (size_t)(nb > 0 ? nb : 1));
  c->skp = (int*)malloc(sizeof(int) * (size_t)(nb > 0 ? nb : 1));
  c->nlag = c->nflx = c->nskp = 0;
  for (int ib = 0; ib < nb; ++ib) {
    int lag_act = c->interior[ib] > 0;
    int flx_act = lag_act || c->halo[ib] > 0;
    if (!c->opt.skip_dry_blocks) {
      c->lag[c->nlag++] = ib;
      c->flx[c->nflx++] = ib;
    } else {
      if (lag_act) c->lag[c->nlag++] = ib;
      if (flx_act) c->flx[c->nflx++] = ib;
      else c->skp[c->nskp++] = ib;
    }
  }
  c->blk_reduce = dalloc(nb);
  c->blk_srcvol = dalloc(nb);
  c->blk_err = (long long*)malloc(sizeof(long long) * (size_t)(nb > 0 ? nb : 1));
  for (int ib = 0; ib < nb; ++ib) c->blk_err[ib] = -1;
}

static int flux_active(const orc_ctx* c, int ib) { return c->interior[ib] > 0 || c->halo[ib] > 0; }

/* begin_step, stepper.cpp:172-201 */
static int begin_step(orc_ctx* c) {
  if (c->nsrc > 0) {
    for (int s = 0; s < c->nsrc; ++s) { /* source_terms re-validates, sources.cpp:50 */
      swf_source tmp = {c->src[s].kind, c->src[s].i0, c->src[s].j0, c->src[s].i1, c->src[s].j1,
                        c->src[s].nh, c->src[s].ht, c->src[s].hq, c->src[s].rate, c->src[s].vx,
                        c->src[s].vy};
      int rc = validate_source(c, &tmp, s);
      if (rc) return rc;
    }
    source_terms(c, c->t);
  }
  compute_block_mask(c);
  c->clamp_deficit = 0.0;
  c->source_volume = 0.0;
  c->boundary_outflow = 0.0;
  return SWF_OK;
}

/* ------------------------------------------------------------------------ */
/* views: the step-start state (detail::StateRef, forcing.hpp:64-71) or the */
/* half-step view (CsphTvdStepper::HalfView, stepper.cpp:54-74)              */
/* ------------------------------------------------------------------------ */

typedef struct {
  const orc_ctx* c;
  int half; /* 0: StateRef, 1: HalfView */
} view;

static inline int v_act(const view* v, size_t k) {
  return v->c->H[k] > v->c->p.eps_dry || v->c->q[k] != 0;
}
static inline double v_depth(const view* v, size_t k) {
  if (v->half && v_act(v, k)) return v->c->hH[k];
  return v->c->H[k];
}
static inline double v_momx(const view* v, size_t k) {
  if (v->half && v_act(v, k)) return v->c->hHUx[k];
  return v->c->HUx[k];
}
static inline double v_momy(const view* v, size_t k) {
  if (v->half && v_act(v, k)) return v->c->hHUy[k];
  return v->c->HUy[k];
}
static inline double v_shiftx(const view* v, size_t k) { return v_act(v, k) ? 0.5 * v->c->drx[k] : 0.0; }
static inline double v_shifty(const view* v, size_t k) { return v_act(v, k) ? 0.5 * v->c->dry[k] : 0.0; }

/* ------------------------------------------------------------------------ */
/* forcing: forcing.hpp:74-237                                               */
/* ------------------------------------------------------------------------ */

/* friction_core, forcing.hpp:80-84 */
static void friction_core(double ux, double uy, double H, double g, double n, double* fx, double* fy) {
  double lam = ((2.0 * g) * n) * n / (H * orc_cbrt(H));
  double speed = sqrt(ux * ux + uy * uy);
  *fx = ((-0.5 * lam) * ux) * speed;
  *fy = ((-0.5 * lam) * uy) * speed;
}

/* eta_gradient_component, forcing.hpp:89-120; kl/kr < 0 = outside */
static double eta_grad_comp(const view* v, double eta_c, long long kl, long long kr) {
  const orc_ctx* c = v->c;
  double eps = c->p.eps_dry, h = c->h;
  int has_l = 0, has_r = 0;
  double eta_l = 0.0, eta_r = 0.0;
  if (kl >= 0) {
    double Hl = v_depth(v, (size_t)kl);
    double el = Hl + c->b[kl];
    if (Hl > eps || el < eta_c) { has_l = 1; eta_l = el; }
  }
  if (kr >= 0) {
    double Hr = v_depth(v, (size_t)kr);
    double er = Hr + c->b[kr];
    if (Hr > eps || er < eta_c) { has_r = 1; eta_r = er; }
  }
  if (has_l && has_r) return (eta_r - eta_l) / (2.0 * h);
  if (has_r) return (eta_r - eta_c) / h;
  if (has_l) return (eta_c - eta_l) / h;
  return 0.0;
}

/* eta_gradient, forcing.hpp:122-135 */
static void eta_gradient(const view* v, int i, int j, double* gx, double* gy) {
  const orc_ctx* c = v->c;
  long long nx = c->nx;
  long long k = i + j * nx;
  double eta_c = v_depth(v, (size_t)k) + c->b[k];
  *gx = eta_grad_comp(v, eta_c, i > 0 ? k - 1 : -1, i + 1 < c->nx ? k + 1 : -1);
  *gy = eta_grad_comp(v, eta_c, j > 0 ? k - nx : -1, j + 1 < c->ny ? k + nx : -1);
}

/* laplacian_velocity, forcing.hpp:137-163 */
static void laplacian(const view* v, int i, int j, double ucx, double ucy, double* lx, double* ly) {
  const orc_ctx* c = v->c;
  double eps = c->p.eps_dry;
  double sx = 0.0, sy = 0.0;
  const int di[4] = {-1, 1, 0, 0}, dj[4] = {0, 0, -1, 1};
  for (int m = 0; m < 4; ++m) {
    int ni = i + di[m], nj = j + dj[m];
    if (ni < 0 || ni >= c->nx || nj < 0 || nj >= c->ny) { sx += ucx; sy += ucy; continue; }
    size_t nk = (size_t)ni + (size_t)nj * c->nx;
    double Hn = v_depth(v, nk);
    if (Hn > eps) {
      /* view_velocity, forcing.hpp:74-78 */
      sx += v_momx(v, nk) / Hn;
      sy += v_momy(v, nk) / Hn;
    } else { sx += ucx; sy += ucy; }
  }
  double inv_h2 = 1.0 / (c->h * c->h);
  *lx = (sx - 4.0 * ucx) * inv_h2;
  *ly = (sy - 4.0 * ucy) * inv_h2;
}

/* assemble_forces_rect, forcing.hpp:177-237, over one block rectangle */
static void assemble_rect(const view* v, double wtx, double wty, int has_wind, const double* sig_arr,
                          int present, double* ofx, double* ofy, double* orx, double* ory, double* osig,
                          int i0, int j0, int i1, int j1) {
  const orc_ctx* c = v->c;
  const swf_params* p = &c->p;
  for (int j = j0; j <= j1; ++j)
    for (int i = i0; i <= i1; ++i) {
      size_t k = (size_t)i + (size_t)j * c->nx;
      double H = v_depth(v, k);
      double sig = present ? sig_arr[k] : 0.0;
      osig[k] = sig;
      if (H <= p->eps_dry) { ofx[k] = 0.0; ofy[k] = 0.0; orx[k] = 0.0; ory[k] = 0.0; continue; }
      double ux = v_momx(v, k) / H, uy = v_momy(v, k) / H;
      double gx, gy;
      eta_gradient(v, i, j, &gx, &gy);
      double fx = -p->g * gx;
      double fy = -p->g * gy;
      double frx, fry;
      friction_core(ux, uy, H, p->g, p->n_field ? p->n_field[k] : p->n_manning, &frx, &fry);
      fx += frx;
      fy += fry;
      if (p->nu > 0.0) {
        double lx, ly;
        laplacian(v, i, j, ux, uy, &lx, &ly);
        fx += p->nu * lx;
        fy += p->nu * ly;
      }
      if (p->omega_z != 0.0) {
        fx += (2.0 * uy) * p->omega_z;
        fy += (-2.0 * ux) * p->omega_z;
      }
      if (has_wind) {
        double rx = wtx - ux, ry = wty - uy;
        double rel = sqrt(rx * rx + ry * ry);
        double cc = (p->c_a * p->rho_air) / (p->rho_water * H);
        fx += (cc * rx) * rel;
        fy += (cc * ry) * rel;
      }
      if (sig != 0.0) {
        double s_h = sig / H;
        fx += s_h * (c->svx[k] - ux);
        fy += s_h * (c->svy[k] - uy);
      }
      ofx[k] = fx; ofy[k] = fy; orx[k] = frx; ory[k] = fry;
    }
}

/* ------------------------------------------------------------------------ */
/* K2 compute_forces, stepper.cpp:210-222                                    */
/* ------------------------------------------------------------------------ */

static void compute_forces(orc_ctx* c) {
  view v = {c, 0};
  double wx, wy;
  wind_at(c, c->t, &wx, &wy);
  for (int n = 0; n < c->nlag; ++n) {
    int i0, j0, i1, j1;
    block_rect(c, c->lag[n], &i0, &j0, &i1, &j1);
    assemble_rect(&v, wx, wy, c->nwind > 0, c->sigma, c->nsrc > 0, c->fn_fx, c->fn_fy, c->fn_rx,
                  c->fn_ry, c->fn_sig, i0, j0, i1, j1);
  }
}

/* ------------------------------------------------------------------------ */
/* K3 compute_dt, stepper.cpp:224-267                                        */
/* ------------------------------------------------------------------------ */

static int compute_dt(orc_ctx* c, double dt_cap, double* tau_out) {
  double eps = c->p.eps_dry, g = c->p.g, h = c->h;
  double speed = 0.0;
  for (int n = 0; n < c->nlag; ++n) {
    int i0, j0, i1, j1;
    block_rect(c, c->lag[n], &i0, &j0, &i1, &j1);
    double m = 0.0;
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) {
        size_t k = (size_t)i + (size_t)j * c->nx;
        double H = c->H[k];
        if (H <= eps) continue;
        double ux = c->HUx[k] / H, uy = c->HUy[k] / H;
        double fx = c->fn_fx[k], fy = c->fn_fy[k];
        double rx = sqrt(h * fabs(fx)), ry = sqrt(h * fabs(fy));
        double upx = fabs(fx > 0.0 ? ux + rx : (fx < 0.0 ? ux - rx : ux));
        double upy = fabs(fy > 0.0 ? uy + ry : (fy < 0.0 ? uy - ry : uy));
        double us = smax(fabs(ux), fabs(uy)) + sqrt(g * H);
        /* std::max({m, up_x, up_y, us}) keeps the first largest */
        double r = m;
        if (r < upx) r = upx;
        if (r < upy) r = upy;
        if (r < us) r = us;
        m = r;
      }
    speed = smax(speed, m);
  }
  double tau = c->ctl.dt_max;
  if (speed > 0.0) {
    double cfl = (c->ctl.courant * h) / speed;
    if (cfl < c->ctl.dt_min)
      return fail(c, SWF_ENUMERICAL,
                  "timestep %f s fell below the abort floor %f s (max wave speed %f m/s)", cfl,
                  c->ctl.dt_min, speed);
    tau = smin(tau, cfl);
  }
  if (dt_cap > 0.0) tau = smin(tau, dt_cap);
  *tau_out = tau;
  return SWF_OK;
}

/* ------------------------------------------------------------------------ */
/* K4 predictor, stepper.cpp:269-308                                         */
/* ------------------------------------------------------------------------ */

static void predictor(orc_ctx* c, double tau) {
  double half_tau = 0.5 * tau, eps = c->p.eps_dry, g = c->p.g;
  for (int n = 0; n < c->nlag; ++n) {
    int i0, j0, i1, j1;
    block_rect(c, c->lag[n], &i0, &j0, &i1, &j1);
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) {
        size_t k = (size_t)i + (size_t)j * c->nx;
        if (!(c->H[k] > eps || c->q[k] != 0)) continue;
        double Hn = c->H[k];
        double H12 = Hn + half_tau * c->sigma[k];
        if (H12 < 0.0) H12 = 0.0;
        double qx = c->HUx[k] + (half_tau * Hn) * (c->fn_fx[k] - c->fn_rx[k]);
        double qy = c->HUy[k] + (half_tau * Hn) * (c->fn_fy[k] - c->fn_ry[k]);
        if (H12 > eps) {
          double nm = c->p.n_field ? c->p.n_field[k] : c->p.n_manning;
          if (nm > 0.0) {
            double ux = qx / H12, uy = qy / H12;
            double sp = sqrt(ux * ux + uy * uy);
            if (sp > 0.0) {
              double lam = ((2.0 * g) * nm) * nm / (H12 * orc_cbrt(H12));
              double fac = 1.0 / (1.0 + ((0.5 * lam) * sp) * half_tau);
              qx = H12 * (ux * fac);
              qy = H12 * (uy * fac);
            }
          }
        } else {
          qx = 0.0;
          qy = 0.0;
        }
        c->hH[k] = H12;
        c->hHUx[k] = qx;
        c->hHUy[k] = qy;
      }
  }
}

/* ------------------------------------------------------------------------ */
/* K5 mid_forces, stepper.cpp:310-333                                        */
/* ------------------------------------------------------------------------ */

static void mid_forces(orc_ctx* c, double tau) {
  double t_mid = c->t + 0.5 * tau;
  if (c->nsrc > 0) resample_sigma(c, t_mid, c->sigma_mid);
  view v = {c, 1};
  double wx, wy;
  wind_at(c, t_mid, &wx, &wy);
  for (int n = 0; n < c->nlag; ++n) {
    int i0, j0, i1, j1;
    block_rect(c, c->lag[n], &i0, &j0, &i1, &j1);
    assemble_rect(&v, wx, wy, c->nwind > 0, c->sigma_mid, c->nsrc > 0, c->fm_fx, c->fm_fy, c->fm_rx,
                  c->fm_ry, c->fm_sig, i0, j0, i1, j1);
  }
}

/* ------------------------------------------------------------------------ */
/* K6 corrector, stepper.cpp:335-400                                         */
/* ------------------------------------------------------------------------ */

static int corrector(orc_ctx* c, double tau) {
  double eps = c->p.eps_dry, g = c->p.g, half_h = 0.5 * c->h;
  int has_src = c->nsrc > 0;
  for (int n = 0; n < c->nlag; ++n) {
    int ib = c->lag[n], i0, j0, i1, j1;
    block_rect(c, ib, &i0, &j0, &i1, &j1);
    double srcvol = 0.0;
    long long err = -1;
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) {
        size_t k = (size_t)i + (size_t)j * c->nx;
        if (!(c->H[k] > eps || c->q[k] != 0)) continue;
        double Hn = c->H[k], Ht = Hn;
        if (has_src) {
          Ht = Hn + tau * c->sigma_mid[k];
          if (Ht < 0.0) Ht = 0.0;
          srcvol += Ht - Hn;
        }
        double H12 = c->hH[k];
        double qx = c->HUx[k] + (tau * H12) * (c->fm_fx[k] - c->fm_rx[k]);
        double qy = c->HUy[k] + (tau * H12) * (c->fm_fy[k] - c->fm_ry[k]);
        if (Ht > eps) {
          double nm = c->p.n_field ? c->p.n_field[k] : c->p.n_manning;
          if (nm > 0.0) {
            double ux = qx / Ht, uy = qy / Ht;
            double sp = sqrt(ux * ux + uy * uy);
            if (sp > 0.0) {
              double lam = ((2.0 * g) * nm) * nm / (Ht * orc_cbrt(Ht));
              double fac = 1.0 / (1.0 + ((0.5 * lam) * sp) * tau);
              qx = Ht * (ux * fac);
              qy = Ht * (uy * fac);
            }
          }
        }
        double ux12 = 0.0, uy12 = 0.0;
        if (H12 > eps) { ux12 = c->hHUx[k] / H12; uy12 = c->hHUy[k] / H12; }
        double dx = tau * ux12, dy = tau * uy12;
        if (err < 0 && (fabs(dx) >= half_h || fabs(dy) >= half_h)) err = (long long)k;
        c->Ht[k] = Ht; c->HVtx[k] = qx; c->HVty[k] = qy;
        c->drx[k] = dx; c->dry[k] = dy;
      }
    c->blk_srcvol[ib] = srcvol;
    c->blk_err[ib] = err;
  }
  for (int n = 0; n < c->nlag; ++n) {
    long long k = c->blk_err[c->lag[n]];
    if (k >= 0)
      return fail(c, SWF_ENUMERICAL,
                  "particle displacement reached h/2 at cell (%lld,%lld); the Courant number is too "
                  "large for this flow",
                  k % c->nx, k / c->nx);
  }
  return SWF_OK;
}

/* ------------------------------------------------------------------------ */
/* K7 flux: stepper.cpp:89-123, 402-626; riemann.cpp:14-64                   */
/* ------------------------------------------------------------------------ */

typedef struct { double fm, fn; } flux1;

/* physical_flux, riemann.cpp:14-17 */
static flux1 phys_flux(double h, double un, double g) {
  double q = h * un;
  flux1 f = {q, q * un + ((0.5 * g) * h) * h};
  return f;
}

/* dry_right_fan, riemann.cpp:20-29 */
static flux1 dry_right_fan(double hL, double unL, double g) {
  double cL = sqrt(g * hL);
  double head = unL - cL;
  double front = unL + 2.0 * cL;
  if (head >= 0.0) return phys_flux(hL, unL, g);
  if (front <= 0.0) { flux1 z = {0.0, 0.0}; return z; }
  double u0 = (unL + 2.0 * cL) / 3.0;
  double h0 = (u0 * u0) / g;
  return phys_flux(h0, u0, g);
}

/* hll_face_flux, riemann.cpp:33-64 */
static void hll(double hL, double unL, double utL, double hR, double unR, double utR, double g,
                double* fm, double* fn, double* ft) {
  int dryL = hL <= 0.0, dryR = hR <= 0.0;
  if (dryL && dryR) { *fm = 0.0; *fn = 0.0; *ft = 0.0; return; }
  flux1 f;
  if (dryR) {
    f = dry_right_fan(hL, unL, g);
  } else if (dryL) {
    flux1 m = dry_right_fan(hR, -unR, g);
    f.fm = -m.fm;
    f.fn = m.fn;
  } else {
    double cL = sqrt(g * hL), cR = sqrt(g * hR);
    double sL = smin(unL - cL, unR - cR);
    double sR = smax(unL + cL, unR + cR);
    flux1 fL = phys_flux(hL, unL, g), fR = phys_flux(hR, unR, g);
    if (sL >= 0.0) f = fL;
    else if (sR <= 0.0) f = fR;
    else {
      double inv = 1.0 / (sR - sL);
      f.fm = ((sR * fL.fm - sL * fR.fm) + (sL * sR) * (hR - hL)) * inv;
      f.fn = ((sR * fL.fn - sL * fR.fn) + (sL * sR) * (hR * unR - hL * unL)) * inv;
    }
  }
  *fm = f.fm;
  *fn = f.fn;
  *ft = f.fm * (f.fm >= 0.0 ? utL : utR);
}

void orc_hll_face_flux(const double* in, double g, double* out) {
  hll(in[0], in[1], in[2], in[3], in[4], in[5], g, &out[0], &out[1], &out[2]);
}

typedef struct { double hs, hcell, un, ut; } side_state; /* SideState, stepper.cpp:78-83 */

/* reconstruct_side, stepper.cpp:89-123.  dir 0 = x faces, 1 = y faces. */
static side_state reconstruct(const view* v, int dir, double b_face, size_t k, long long kout,
                              size_t kin, double sgn) {
  const orc_ctx* c = v->c;
  double eps = c->p.eps_dry, h = c->h;
  side_state s = {0.0, 0.0, 0.0, 0.0};
#define SHIFT(kk) (dir == 0 ? v_shiftx(v, (kk)) : v_shifty(v, (kk)))
#define UN(kk) (v_depth(v, (kk)) > eps ? (dir == 0 ? v_momx(v, (kk)) : v_momy(v, (kk))) / v_depth(v, (kk)) : 0.0)
#define UT(kk) (v_depth(v, (kk)) > eps ? (dir == 0 ? v_momy(v, (kk)) : v_momx(v, (kk))) / v_depth(v, (kk)) : 0.0)
  double eta_c = v_depth(v, k) + c->b[k];
  double un_c = UN(k), ut_c = UT(k);
  double p_c = SHIFT(k);
  double p_in = sgn * h + SHIFT(kin);
  double face = (sgn * 0.5) * h;
  double s_eta = 0.0, s_un = 0.0, s_ut = 0.0;
  if (kout >= 0) {
    size_t ko = (size_t)kout;
    double p_out = -sgn * h + SHIFT(ko);
    double d_in = p_in - p_c, d_out = p_c - p_out;
    s_eta = minmod(((v_depth(v, kin) + c->b[kin]) - eta_c) / d_in,
                   (eta_c - (v_depth(v, ko) + c->b[ko])) / d_out);
    s_un = minmod((UN(kin) - un_c) / d_in, (un_c - UN(ko)) / d_out);
    s_ut = minmod((UT(kin) - ut_c) / d_in, (ut_c - UT(ko)) / d_out);
  }
#undef SHIFT
#undef UN
#undef UT
  double off = face - p_c;
  double eta_f = eta_c + s_eta * off;
  s.hcell = smax(0.0, eta_f - c->b[k]);
  if (s.hcell <= 0.0) { s.hcell = 0.0; return s; }
  s.hs = smax(0.0, eta_f - b_face);
  s.un = un_c + s_un * off;
  s.ut = ut_c + s_ut * off;
  return s;
}

static int v_wet(const view* v, size_t k) { return v_depth(v, k) > v->c->p.eps_dry; }

static face_rec make_face(const view* v, int dir, size_t ka, size_t kb, long long kouta, long long koutb) {
  const orc_ctx* c = v->c;
  face_rec rec = {0.0, 0.0, 0.0, 0.0};
  int wetA = v_wet(v, ka), wetB = v_wet(v, kb);
  if (!wetA && !wetB) return rec;
  double g = c->p.g;
  double bf = smax(c->b[ka], c->b[kb]);
  side_state L = {0.0, 0.0, 0.0, 0.0}, R = {0.0, 0.0, 0.0, 0.0};
  if (wetA) L = reconstruct(v, dir, bf, ka, kouta, kb, 1.0);
  if (wetB) R = reconstruct(v, dir, bf, kb, koutb, ka, -1.0);
  double fm, fn, ft;
  hll(L.hs, L.un, L.ut, R.hs, R.un, R.ut, g, &fm, &fn, &ft);
  rec.fm = fm;
  rec.ft = ft;
  rec.fnl = (fn - ((0.5 * g) * L.hs) * L.hs) + ((0.5 * g) * L.hcell) * L.hcell;
  rec.fnr = (fn - ((0.5 * g) * R.hs) * R.hs) + ((0.5 * g) * R.hcell) * R.hcell;
  return rec;
}

/* compute_x_face, stepper.cpp:402-447 */
static void x_face(orc_ctx* c, const view* v, int iface, int j) {
  size_t nx = c->nx;
  size_t ka = (size_t)(iface - 1) + j * nx, kb = (size_t)iface + j * nx;
  face_rec rec = make_face(v, 0, ka, kb, iface - 2 >= 0 ? (long long)ka - 1 : -1,
                           iface + 1 < c->nx ? (long long)kb + 1 : -1);
  if (!isfinite(rec.fm + rec.fnl + rec.fnr + rec.ft)) {
    int ib = (iface == c->nx ? c->nx - 1 : iface) / c->bs + (j / c->bs) * c->nbx;
    c->blk_err[ib] = (long long)ka;
  }
  c->xf[(size_t)iface + (size_t)j * (nx + 1)] = rec;
}

/* compute_y_face, stepper.cpp:449-494 */
static void y_face(orc_ctx* c, const view* v, int i, int jface) {
  size_t nx = c->nx;
  size_t ka = (size_t)i + (size_t)(jface - 1) * nx, kb = (size_t)i + (size_t)jface * nx;
  face_rec rec = make_face(v, 1, ka, kb, jface - 2 >= 0 ? (long long)(ka - nx) : -1,
                           jface + 1 < c->ny ? (long long)(kb + nx) : -1);
  if (!isfinite(rec.fm + rec.fnl + rec.fnr + rec.ft)) {
    int ib = i / c->bs + ((jface == c->ny ? c->ny - 1 : jface) / c->bs) * c->nbx;
    c->blk_err[ib] = (long long)ka;
  }
  c->yf[(size_t)i + (size_t)jface * nx] = rec;
}

/* boundary_x_face / boundary_y_face, stepper.cpp:496-538 */
static void bnd_face(orc_ctx* c, const view* v, int dir, int a, int faceidx) {
  size_t nx = c->nx;
  face_rec rec = {0.0, 0.0, 0.0, 0.0};
  int lo = (faceidx == 0);
  size_t k;
  int kind;
  if (dir == 0) {
    k = lo ? (size_t)a * nx : (size_t)(c->nx - 1) + (size_t)a * nx;
    kind = lo ? c->opt.west : c->opt.east;
  } else {
    k = lo ? (size_t)a : (size_t)a + (size_t)(c->ny - 1) * nx;
    kind = lo ? c->opt.south : c->opt.north;
  }
  if (v_wet(v, k)) {
    double H = v_depth(v, k);
    double ux = v_momx(v, k) / H, uy = v_momy(v, k) / H;
    double un = dir == 0 ? ux : uy, ut = dir == 0 ? uy : ux;
    double ghost = (kind == SWF_EDGE_REFLECTIVE) ? -un : un;
    double fm, fn, ft;
    if (lo) hll(H, ghost, ut, H, un, ut, c->p.g, &fm, &fn, &ft);
    else hll(H, un, ut, H, ghost, ut, c->p.g, &fm, &fn, &ft);
    rec.fm = fm; rec.fnl = fn; rec.fnr = fn; rec.ft = ft;
  }
  if (dir == 0) c->xf[(size_t)faceidx + (size_t)a * (nx + 1)] = rec;
  else c->yf[(size_t)a + (size_t)faceidx * nx] = rec;
}

/* accumulate_cell, stepper.cpp:540-566 */
static void accumulate(orc_ctx* c, const view* v, int i, int j) {
  size_t nx = c->nx;
  size_t k = (size_t)i + (size_t)j * nx;
  const face_rec* W = &c->xf[(size_t)i + (size_t)j * (nx + 1)];
  const face_rec* E = &c->xf[(size_t)i + 1 + (size_t)j * (nx + 1)];
  const face_rec* S = &c->yf[(size_t)i + (size_t)j * nx];
  const face_rec* N = &c->yf[(size_t)i + (size_t)(j + 1) * nx];
  c->Fh[k] = (W->fm - E->fm) + (S->fm - N->fm);
  double cx = 0.0, cy = 0.0;
  if (v_wet(v, k)) {
    double gx, gy;
    eta_gradient(v, i, j, &gx, &gy);
    double gh = (c->p.g * v_depth(v, k)) * c->h;
    cx = gh * gx;
    cy = gh * gy;
  }
  c->Fvx[k] = ((W->fnr - E->fnl) + (S->ft - N->ft)) + cx;
  c->Fvy[k] = ((S->fnr - N->fnl) + (W->ft - E->ft)) + cy;
}

/* flux, stepper.cpp:579-626 */
static int flux(orc_ctx* c) {
  view v = {c, 1};
  int skip = c->opt.skip_dry_blocks;
  for (int n = 0; n < c->nflx; ++n) {
    int ib = c->flx[n], i0, j0, i1, j1;
    block_rect(c, ib, &i0, &j0, &i1, &j1);
    int bi = ib % c->nbx, bj = ib / c->nbx;
    int own_west = (bi == 0) || (skip && !flux_active(c, ib - 1));
    int own_south = (bj == 0) || (skip && !flux_active(c, ib - c->nbx));
    for (int j = j0; j <= j1; ++j) {
      if (own_west) {
        if (i0 == 0) bnd_face(c, &v, 0, j, 0);
        else x_face(c, &v, i0, j);
      }
      for (int f = i0 + 1; f <= i1; ++f) x_face(c, &v, f, j);
      if (i1 + 1 == c->nx) bnd_face(c, &v, 0, j, c->nx);
      else x_face(c, &v, i1 + 1, j);
    }
    for (int i = i0; i <= i1; ++i) {
      if (own_south) {
        if (j0 == 0) bnd_face(c, &v, 1, i, 0);
        else y_face(c, &v, i, j0);
      }
      for (int f = j0 + 1; f <= j1; ++f) y_face(c, &v, i, f);
      if (j1 + 1 == c->ny) bnd_face(c, &v, 1, i, c->ny);
      else y_face(c, &v, i, j1 + 1);
    }
  }
  /* raise_pending_error, stepper.cpp:568-577 */
  for (int n = 0; n < c->nflx; ++n) {
    long long k = c->blk_err[c->flx[n]];
    if (k >= 0)
      return fail(c, SWF_ENUMERICAL, "non-finite flux near cell (%lld,%lld)", k % c->nx, k / c->nx);
  }
  for (int n = 0; n < c->nflx; ++n) {
    int i0, j0, i1, j1;
    block_rect(c, c->flx[n], &i0, &j0, &i1, &j1);
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) accumulate(c, &v, i, j);
  }
  return SWF_OK;
}

/* ------------------------------------------------------------------------ */
/* K8 final_update, stepper.cpp:628-704                                      */
/* ------------------------------------------------------------------------ */

static void final_update(orc_ctx* c, double tau) {
  double dt_h = tau / c->h, eps = c->p.eps_dry;
  size_t nx = c->nx;
  for (int n = 0; n < c->nflx; ++n) {
    int ib = c->flx[n], i0, j0, i1, j1;
    block_rect(c, ib, &i0, &j0, &i1, &j1);
    double deficit = 0.0;
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) {
        size_t k = (size_t)i + (size_t)j * nx;
        int act = c->H[k] > eps || c->q[k] != 0;
        double base = act ? c->Ht[k] : c->H[k];
        double Hn1 = base + dt_h * c->Fh[k];
        if (Hn1 < 0.0) { deficit += -Hn1; Hn1 = 0.0; }
        double qx = 0.0, qy = 0.0;
        if (Hn1 > eps) {
          qx = (act ? c->HVtx[k] : c->HUx[k]) + dt_h * c->Fvx[k];
          qy = (act ? c->HVty[k] : c->HUy[k]) + dt_h * c->Fvy[k];
        }
        c->H[k] = Hn1; c->HUx[k] = qx; c->HUy[k] = qy;
        c->Ht[k] = 0.0; c->HVtx[k] = 0.0; c->HVty[k] = 0.0;
      }
    c->blk_reduce[ib] = deficit;
  }
  for (int n = 0; n < c->nskp; ++n) {
    int i0, j0, i1, j1;
    block_rect(c, c->skp[n], &i0, &j0, &i1, &j1);
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) {
        size_t k = (size_t)i + (size_t)j * nx;
        c->Ht[k] = 0.0; c->HVtx[k] = 0.0; c->HVty[k] = 0.0;
      }
  }
  double area = c->h * c->h;
  double deficit = 0.0;
  for (int n = 0; n < c->nflx; ++n) deficit += c->blk_reduce[c->flx[n]];
  c->clamp_deficit = deficit * area;
  double srcvol = 0.0;
  for (int n = 0; n < c->nlag; ++n) srcvol += c->blk_srcvol[c->lag[n]];
  c->source_volume = srcvol * area;
  /* net outflow through domain edges, stepper.cpp:684-701 */
  double out = 0.0;
#define LIVE(ci, cj) (!c->opt.skip_dry_blocks || flux_active(c, (ci) / c->bs + ((cj) / c->bs) * c->nbx))
  for (int j = 0; j < c->ny; ++j) {
    if (LIVE(0, j)) out -= c->xf[(size_t)j * (nx + 1)].fm;
    if (LIVE(c->nx - 1, j)) out += c->xf[(size_t)c->nx + (size_t)j * (nx + 1)].fm;
  }
  for (int i = 0; i < c->nx; ++i) {
    if (LIVE(i, 0)) out -= c->yf[i].fm;
    if (LIVE(i, c->ny - 1)) out += c->yf[(size_t)i + (size_t)c->ny * nx].fm;
  }
#undef LIVE
  c->boundary_outflow = (out * tau) * c->h;
  c->t += tau;
}

/* ------------------------------------------------------------------------ */
/* step, stepper.cpp:706-749, and the stage interface                        */
/* ------------------------------------------------------------------------ */

int orc_stage(orc_ctx* c, int stage, double arg, double* tau_out) {
  switch (stage) {
    case SWF_STAGE_BEGIN: return begin_step(c);
    case SWF_STAGE_FORCES: compute_forces(c); return SWF_OK;
    case SWF_STAGE_DT: {
      double tau = 0.0;
      int rc = compute_dt(c, arg, &tau);
      if (rc == SWF_OK && tau_out) *tau_out = tau;
      return rc;
    }
    case SWF_STAGE_PREDICTOR: predictor(c, arg); return SWF_OK;
    case SWF_STAGE_MID_FORCES: mid_forces(c, arg); return SWF_OK;
    case SWF_STAGE_CORRECTOR: return corrector(c, arg);
    case SWF_STAGE_FLUX: return flux(c);
    case SWF_STAGE_FINAL: final_update(c, arg); return SWF_OK;
    default: return fail(c, SWF_ECONFIG, "unknown stage id");
  }
}

int orc_step(orc_ctx* c, double dt_cap, swf_step_info* info) {
  int rc;
  double tau = 0.0;
  if ((rc = begin_step(c))) return rc;
  compute_forces(c);
  if ((rc = compute_dt(c, dt_cap, &tau))) return rc;
  predictor(c, tau);
  mid_forces(c, tau);
  if ((rc = corrector(c, tau))) return rc;
  if ((rc = flux(c))) return rc;
  final_update(c, tau);
  if (info) {
    memset(info, 0, sizeof *info);
    info->tau = tau;
    int nb = c->nbx * c->nby, act = 0;
    for (int ib = 0; ib < nb; ++ib) act += flux_active(c, ib);
    info->active_fraction = nb ? (double)act / nb : 0.0;
    info->lagrangian_blocks = c->nlag;
    info->flux_blocks = c->nflx;
    info->total_blocks = nb;
    info->clamp_deficit_volume = c->clamp_deficit;
    info->source_volume = c->source_volume;
    info->boundary_outflow_volume = c->boundary_outflow;
  }
  return SWF_OK;
}

int orc_run(orc_ctx* c, int n, double dt_cap, int* done, swf_step_info* last) {
  if (done) *done = 0;
  for (int k = 0; k < n; ++k) {
    int rc = orc_step(c, dt_cap, last);
    if (rc) return rc;
    if (done) *done = k + 1;
  }
  return SWF_OK;
}

/* ------------------------------------------------------------------------ */
/* accessors                                                                 */
/* ------------------------------------------------------------------------ */

int orc_scratch(orc_ctx* c, int which, double* out) {
  const double* src = NULL;
  switch (which) {
    case SWF_SCR_FN_FX: src = c->fn_fx; break;
    case SWF_SCR_FN_FY: src = c->fn_fy; break;
    case SWF_SCR_FN_FRIC_X: src = c->fn_rx; break;
    case SWF_SCR_FN_FRIC_Y: src = c->fn_ry; break;
    case SWF_SCR_FN_SIGMA: src = c->fn_sig; break;
    case SWF_SCR_FM_FX: src = c->fm_fx; break;
    case SWF_SCR_FM_FY: src = c->fm_fy; break;
    case SWF_SCR_FM_FRIC_X: src = c->fm_rx; break;
    case SWF_SCR_FM_FRIC_Y: src = c->fm_ry; break;
    case SWF_SCR_FM_SIGMA: src = c->fm_sig; break;
    case SWF_SCR_HALF_H: src = c->hH; break;
    case SWF_SCR_HALF_HUX: src = c->hHUx; break;
    case SWF_SCR_HALF_HUY: src = c->hHUy; break;
    case SWF_SCR_HT: src = c->Ht; break;
    case SWF_SCR_HVTX: src = c->HVtx; break;
    case SWF_SCR_HVTY: src = c->HVty; break;
    case SWF_SCR_DRX: src = c->drx; break;
    case SWF_SCR_DRY: src = c->dry; break;
    case SWF_SCR_FH: src = c->Fh; break;
    case SWF_SCR_FVX: src = c->Fvx; break;
    case SWF_SCR_FVY: src = c->Fvy; break;
    case SWF_SCR_SIGMA: src = c->sigma; break;
    case SWF_SCR_SRC_VX: src = c->svx; break;
    case SWF_SCR_SRC_VY: src = c->svy; break;
    default: return fail(c, SWF_ECONFIG, "unknown scratch id");
  }
  memcpy(out, src, cells(c) * sizeof(double));
  return SWF_OK;
}

/* Mass fluxes fm of the faces of the last flux stage (stepper.cpp:402-538):
 * dir 0 = x-faces, (nx+1)*ny values, face i between cells i-1 and i of row j
 * at out[i + j*(nx+1)]; dir 1 = y-faces, nx*(ny+1) values.  Entries of faces
 * the last step did not compute (both adjacent blocks inactive) are stale:
 * callers mask them with orc_mask (their true flux is 0). */
int orc_face_fm(orc_ctx* c, int dir, double* out) {
  size_t n = dir == 0 ? (size_t)(c->nx + 1) * c->ny : (size_t)c->nx * (c->ny + 1);
  const face_rec* f = dir == 0 ? c->xf : c->yf;
  for (size_t k = 0; k < n; ++k) out[k] = f[k].fm;
  return SWF_OK;
}

int orc_mask(orc_ctx* c, int* interior, int* halo, int* nbx, int* nby) {
  if (nbx) *nbx = c->nbx;
  if (nby) *nby = c->nby;
  size_t nb = (size_t)c->nbx * c->nby;
  if (interior && c->interior) memcpy(interior, c->interior, nb * sizeof(int));
  if (halo && c->halo) memcpy(halo, c->halo, nb * sizeof(int));
  return SWF_OK;
}

int orc_volumes(orc_ctx* c, double* cd, double* sv, double* bo) {
  if (cd) *cd = c->clamp_deficit;
  if (sv) *sv = c->source_volume;
  if (bo) *bo = c->boundary_outflow;
  return SWF_OK;
}

/* ------------------------------------------------------------------------ */
/* free functions: forcing.cpp:26-62, grid.cpp:53-56,117-121                  */
/* ------------------------------------------------------------------------ */

void orc_bottom_friction(double ux, double uy, double H, double g, double n, double* out) {
  friction_core(ux, uy, H, g, n, &out[0], &out[1]);
}

void orc_coriolis_force(double ux, double uy, double omega_z, double* out) {
  out[0] = (2.0 * uy) * omega_z;
  out[1] = (-2.0 * ux) * omega_z;
}

void orc_wind_force(double ux, double uy, double H, double wx, double wy, double c_a,
                    double rho_air, double rho_water, double* out) {
  double rx = wx - ux, ry = wy - uy;
  double rel = sqrt(rx * rx + ry * ry);
  double cc = (c_a * rho_air) / (rho_water * H);
  out[0] = (cc * rx) * rel;
  out[1] = (cc * ry) * rel;
}

static orc_ctx* temp_ctx(const swf_terrain* T, const swf_params* P, const double* H,
                         const double* HUx, const double* HUy) {
  orc_ctx* c = (orc_ctx*)calloc(1, sizeof *c);
  c->nx = T->nx; c->ny = T->ny; c->h = T->h;
  c->b = (double*)T->b;
  c->p = *P;
  c->H = (double*)H; c->HUx = (double*)HUx; c->HUy = (double*)HUy;
  c->q = (uint8_t*)calloc(cells(c), 1);
  return c;
}

int orc_viscous_force(const swf_terrain* T, const swf_params* P, const double* H,
                      const double* HUx, const double* HUy, int i, int j, double* out) {
  if (i < 0 || i >= T->nx || j < 0 || j >= T->ny) return fail(NULL, SWF_ERANGE, "cell index outside grid");
  orc_ctx* c = temp_ctx(T, P, H, HUx, HUy);
  view v = {c, 0};
  size_t k = (size_t)i + (size_t)j * T->nx;
  double ux = 0.0, uy = 0.0, lx, ly;
  if (H[k] > P->eps_dry) { ux = HUx[k] / H[k]; uy = HUy[k] / H[k]; }
  laplacian(&v, i, j, ux, uy, &lx, &ly);
  out[0] = P->nu * lx;
  out[1] = P->nu * ly;
  free(c->q);
  free(c);
  return SWF_OK;
}

int orc_surface_gradient_force(const swf_terrain* T, const swf_params* P, const double* H,
                               const double* HUx, const double* HUy, int i, int j, double* out) {
  if (i < 0 || i >= T->nx || j < 0 || j >= T->ny) return fail(NULL, SWF_ERANGE, "cell index outside grid");
  size_t k = (size_t)i + (size_t)j * T->nx;
  if (H[k] <= P->eps_dry) { out[0] = 0.0; out[1] = 0.0; return SWF_OK; }
  orc_ctx* c = temp_ctx(T, P, H, HUx, HUy);
  view v = {c, 0};
  double gx, gy;
  eta_gradient(&v, i, j, &gx, &gy);
  out[0] = -P->g * gx;
  out[1] = -P->g * gy;
  free(c->q);
  free(c);
  return SWF_OK;
}

double orc_total_volume(int n, const double* H, double h) {
  double sum = 0.0;
  for (int k = 0; k < n; ++k) sum += H[k];
  return sum * (h * h);
}

double orc_latitude_to_omega_z(double lat) {
  return 7.2921159e-5 * sin(lat * 3.141592653589793 / 180.0);
}
