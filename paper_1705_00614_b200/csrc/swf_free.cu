// swf_free.cu — the reference's free functions of the step's data path,
// evaluated on the device (C ABI in include/swf.h, C++ wrappers in
// host/swflood_b200.cpp):
//   forcing.hpp:34-57  viscous_force, coriolis_force, wind_force,
//                      surface_gradient_force, assemble_forces
//   block.hpp:38-39    compute_block_mask
//   sources.hpp:40-46  source_terms, resample_sigma
// Every per-cell expression is the one the step kernels use (swf_math.cuh),
// exact (no speculative forms), so the results equal the reference's bit for
// bit (tests/test_free_functions.py; tests/native/dropin_free_test.cpp).
// Citations are relative to /root/reference/proj.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "swf_internal.cuh"

namespace swf {
namespace {

constexpr int FT = 256;

PhysConst phys_of(const swf_terrain* T, const swf_params* P) {
  PhysConst c;
  c.g = P->g;
  c.nu = P->nu;
  c.omega_z = P->omega_z;
  c.c_a = P->c_a;
  c.rho_air = P->rho_air;
  c.rho_water = P->rho_water;
  c.eps = P->eps_dry;
  c.h = T->h;
  c.inv_h2 = 1.0 / (T->h * T->h);  // forcing.hpp:161
  c.two_h = 2.0 * T->h;            // forcing.hpp:116
  // r = 0: rdiv falls back to the plain (correctly rounded) division
  c.rh.b = T->h;
  c.rh.r = 0.0;
  c.r2h.b = c.two_h;
  c.r2h.r = 0.0;
  return c;
}

// StateRef (forcing.hpp:64-71) over device arrays
struct DState {
  const double *H, *HUx, *HUy, *b;
  int nx, ny;
  double eps;
  __device__ Nbr nbr(bool in, size_t k) const {
    Nbr n;
    n.in = in;
    n.depth = n.eta = n.ux = n.uy = 0.0;
    if (in) {
      n.depth = H[k];
      n.eta = n.depth + b[k];
      if (n.depth > eps) {  // view_velocity, forcing.hpp:74-78
        n.ux = HUx[k] / n.depth;
        n.uy = HUy[k] / n.depth;
      }
    }
    return n;
  }
};

// assemble_forces (forcing.cpp:58-70 -> assemble_forces_rect, forcing.hpp:177-237)
// over every cell; sigma == nullptr: no sources (src.empty()).
__global__ void k_assemble(DState v, PhysConst P, double n_manning, const double* nf,
                           bool has_wind, double wx, double wy, const double* sigma,
                           const double* svx, const double* svy, double* fx, double* fy,
                           double* frx, double* fry, double* fsig) {
  size_t k = (size_t)blockIdx.x * FT + threadIdx.x;
  const size_t n = (size_t)v.nx * v.ny;
  if (k >= n) return;
  const int i = (int)(k % v.nx), j = (int)(k / v.nx);
  const double H = v.H[k];
  const double sig = sigma ? sigma[k] : 0.0;
  fsig[k] = sig;
  if (H <= P.eps) {
    fx[k] = fy[k] = frx[k] = fry[k] = 0.0;
    return;
  }
  const double ux = v.HUx[k] / H, uy = v.HUy[k] / H;
  const size_t nx = v.nx;
  Nbr W = v.nbr(i > 0, k - 1), E = v.nbr(i + 1 < v.nx, k + 1);
  Nbr S = v.nbr(j > 0, k - nx), N = v.nbr(j + 1 < v.ny, k + nx);
  ForceOut o = cell_forces(H, ux, uy, H + v.b[k], W, E, S, N, nf ? nf[k] : n_manning, P, has_wind,
                           wx, wy, sig, sigma ? svx[k] : 0.0, sigma ? svy[k] : 0.0);
  fx[k] = o.fx;
  fy[k] = o.fy;
  frx[k] = o.frx;
  fry[k] = o.fry;
}

// viscous_force (forcing.cpp:34-40, which = 0) and surface_gradient_force
// (forcing.cpp:54-60, which = 1) at listed cells
__global__ void k_point_forces(DState v, PhysConst P, int which, int npt, const int* ij,
                               double* out) {
  int q = blockIdx.x * FT + threadIdx.x;
  if (q >= npt) return;
  const int i = ij[2 * q], j = ij[2 * q + 1];
  const size_t k = (size_t)i + (size_t)j * v.nx, nx = v.nx;
  Nbr W = v.nbr(i > 0, k - 1), E = v.nbr(i + 1 < v.nx, k + 1);
  Nbr S = v.nbr(j > 0, k - nx), N = v.nbr(j + 1 < v.ny, k + nx);
  const Nbr C = v.nbr(true, k);
  double rx = 0.0, ry = 0.0;
  if (which == 0) {
    double lx, ly;
    laplacian(W, E, S, N, C.ux, C.uy, P, lx, ly);  // u_c = view_velocity (0 when dry)
    rx = P.nu * lx;
    ry = P.nu * ly;
  } else if (C.depth > P.eps) {
    double gx = eta_grad_comp(W, E, C.eta, P);
    double gy = eta_grad_comp(S, N, C.eta, P);
    rx = -P.g * gx;
    ry = -P.g * gy;
  }
  out[2 * (size_t)q] = rx;
  out[2 * (size_t)q + 1] = ry;
}

// coriolis_force (forcing.cpp:42-44): in = n x {ux, uy}
__global__ void k_coriolis(int n, const double* u, double omega_z, double* out) {
  int q = blockIdx.x * FT + threadIdx.x;
  if (q >= n) return;
  out[2 * (size_t)q] = (2.0 * u[2 * (size_t)q + 1]) * omega_z;
  out[2 * (size_t)q + 1] = (-2.0 * u[2 * (size_t)q]) * omega_z;
}

// wind_force (forcing.cpp:46-52) with W already sampled: in = n x {ux, uy, H}
__global__ void k_wind(int n, const double* in, double wx, double wy, PhysConst P, double* out) {
  int q = blockIdx.x * FT + threadIdx.x;
  if (q >= n) return;
  const double ux = in[3 * (size_t)q], uy = in[3 * (size_t)q + 1], H = in[3 * (size_t)q + 2];
  const double rx = wx - ux, ry = wy - uy;
  const double rel = sqrt(rx * rx + ry * ry);
  const double c = (P.c_a * P.rho_air) / (P.rho_water * H);
  out[2 * (size_t)q] = (c * rx) * rel;
  out[2 * (size_t)q + 1] = (c * ry) * rel;
}

// compute_block_mask (block.cpp:16-61): one thread per block; interior cells
// and the one-cell ring with positions clamped into the domain
__global__ void k_block_mask(int nx, int ny, const double* H, const unsigned char* q, double eps,
                             int bs, int nbx, int nby, int* interior, int* halo) {
  int ib = blockIdx.x * FT + threadIdx.x;
  if (ib >= nbx * nby) return;
  const int i0 = (ib % nbx) * bs, j0 = (ib / nbx) * bs;
  const int i1 = min(i0 + bs - 1, nx - 1), j1 = min(j0 + bs - 1, ny - 1);
  auto wet = [&](int i, int j) {
    size_t k = (size_t)i + (size_t)j * nx;
    return H[k] > eps || (q && q[k] != 0);
  };
  int in = 0;
  for (int j = j0; j <= j1; ++j)
    for (int i = i0; i <= i1; ++i) in += wet(i, j);
  int ring = 0;
  auto at = [&](int i, int j) { ring += wet(min(max(i, 0), nx - 1), min(max(j, 0), ny - 1)); };
  for (int i = i0 - 1; i <= i1 + 1; ++i) {
    at(i, j0 - 1);
    at(i, j1 + 1);
  }
  for (int j = j0; j <= j1; ++j) {
    at(i0 - 1, j);
    at(i1 + 1, j);
  }
  interior[ib] = in;
  halo[ib] = ring;
}

// per-spec sigma at t (cell_sigma, sources.cpp:37-41)
__global__ void k_spec_sigma(const DevSrc* src, int ns, const double* ht, const double* hq,
                             double t, double* sig) {
  int m = blockIdx.x * FT + threadIdx.x;
  if (m >= ns) return;
  const DevSrc& d = src[m];
  sig[m] = d.kind == SWF_SOURCE_RAIN ? d.rate
                                      : series_at(ht + d.off, hq + d.off, d.nh, 1, 0, t) / d.count_area;
}

// source_terms (sources.cpp:43-64; resample = 0) and resample_sigma
// (sources.cpp:66-75; resample = 1: sigma only, markers and velocities kept):
// per cell, the covering specs summed in spec order, the last one's velocity
__global__ void k_source_fill(int nx, int ny, const DevSrc* src, int ns, const double* sig,
                              int resample, double* sigma, double* vx, double* vy,
                              unsigned char* q) {
  size_t k = (size_t)blockIdx.x * FT + threadIdx.x;
  if (k >= (size_t)nx * ny) return;
  const int i = (int)(k % nx), j = (int)(k / nx);
  double svx = resample ? 0.0 : vx[k], svy = resample ? 0.0 : vy[k];
  const double s = cell_source(src, sig, ns, i, j, svx, svy);
  sigma[k] = s;
  if (!resample) {
    vx[k] = svx;
    vy[k] = svy;
    q[k] = s != 0.0 ? 1 : 0;
  }
}

// device buffers of one call, freed on every return path
struct Bufs {
  std::vector<void*> p;
  ~Bufs() {
    for (void* q : p) cudaFree(q);
  }
  template <class T>
  cudaError_t alloc(T** out, size_t n) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, (n ? n : 1) * sizeof(T));
    if (e == cudaSuccess) p.push_back(q);
    *out = (T*)q;
    return e;
  }
  template <class T>
  cudaError_t up(T** out, const T* host, size_t n) {
    cudaError_t e = alloc(out, n);
    if (e == cudaSuccess && n) e = cudaMemcpy(*out, host, n * sizeof(T), cudaMemcpyHostToDevice);
    return e;
  }
};

unsigned nblk(size_t n) { return (unsigned)((n + FT - 1) / FT); }

int grid_ok(const swf_terrain* T) {
  if (!T || T->nx <= 0 || T->ny <= 0) return set_err(nullptr, SWF_ECONFIG, "grid dimensions must be positive");
  return SWF_OK;
}

}  // namespace
}  // namespace swf

using namespace swf;

extern "C" {

int swf_dev_assemble_forces(const swf_terrain* T, const swf_params* P, const double* H,
                            const double* HUx, const double* HUy, int has_wind, double wx,
                            double wy, const double* sigma, const double* svx, const double* svy,
                            double* fx, double* fy, double* fric_x, double* fric_y,
                            double* sigma_eff) {
  if (int rc = grid_ok(T)) return rc;
  const size_t n = (size_t)T->nx * T->ny;
  Bufs B;
  double *dH, *dU, *dV, *db, *dnf = nullptr, *ds = nullptr, *dsx = nullptr, *dsy = nullptr;
  double* o[5];
  cudaError_t e = B.up(&dH, H, n);
  if (e == cudaSuccess) e = B.up(&dU, HUx, n);
  if (e == cudaSuccess) e = B.up(&dV, HUy, n);
  if (e == cudaSuccess) e = B.up(&db, T->b, n);
  if (e == cudaSuccess && P->n_field) e = B.up(&dnf, P->n_field, n);
  if (e == cudaSuccess && sigma) e = B.up(&ds, sigma, n);
  if (e == cudaSuccess && sigma) e = B.up(&dsx, svx, n);
  if (e == cudaSuccess && sigma) e = B.up(&dsy, svy, n);
  for (int m = 0; m < 5 && e == cudaSuccess; ++m) e = B.alloc(&o[m], n);
  if (e == cudaSuccess) {
    DState v{dH, dU, dV, db, T->nx, T->ny, P->eps_dry};
    k_assemble<<<nblk(n), FT>>>(v, phys_of(T, P), P->n_manning, dnf, has_wind != 0, wx, wy, ds,
                                dsx, dsy, o[0], o[1], o[2], o[3], o[4]);
    e = cudaGetLastError();
  }
  double* dst[5] = {fx, fy, fric_x, fric_y, sigma_eff};
  for (int m = 0; m < 5 && e == cudaSuccess; ++m)
    if (dst[m]) e = cudaMemcpy(dst[m], o[m], n * sizeof(double), cudaMemcpyDeviceToHost);
  return cuda_check(nullptr, e, "assemble_forces");
}

int swf_dev_point_forces(const swf_terrain* T, const swf_params* P, const double* H,
                         const double* HUx, const double* HUy, int which, int npt, const int* ij,
                         double* out) {
  if (int rc = grid_ok(T)) return rc;
  for (int q = 0; q < npt; ++q)
    if (ij[2 * q] < 0 || ij[2 * q] >= T->nx || ij[2 * q + 1] < 0 || ij[2 * q + 1] >= T->ny)
      return set_err(nullptr, SWF_ERANGE, "cell index out of range");
  const size_t n = (size_t)T->nx * T->ny;
  Bufs B;
  double *dH, *dU, *dV, *db, *dout;
  int* dij;
  cudaError_t e = B.up(&dH, H, n);
  if (e == cudaSuccess) e = B.up(&dU, HUx, n);
  if (e == cudaSuccess) e = B.up(&dV, HUy, n);
  if (e == cudaSuccess) e = B.up(&db, T->b, n);
  if (e == cudaSuccess) e = B.up(&dij, ij, 2 * (size_t)npt);
  if (e == cudaSuccess) e = B.alloc(&dout, 2 * (size_t)npt);
  if (e == cudaSuccess && npt > 0) {
    DState v{dH, dU, dV, db, T->nx, T->ny, P->eps_dry};
    k_point_forces<<<nblk(npt), FT>>>(v, phys_of(T, P), which, npt, dij, dout);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && npt > 0)
    e = cudaMemcpy(out, dout, 2 * (size_t)npt * sizeof(double), cudaMemcpyDeviceToHost);
  return cuda_check(nullptr, e, which == 0 ? "viscous_force" : "surface_gradient_force");
}

int swf_dev_coriolis_force(int n, const double* u, double omega_z, double* out) {
  Bufs B;
  double *du, *dout;
  cudaError_t e = B.up(&du, u, 2 * (size_t)n);
  if (e == cudaSuccess) e = B.alloc(&dout, 2 * (size_t)n);
  if (e == cudaSuccess && n > 0) {
    k_coriolis<<<nblk(n), FT>>>(n, du, omega_z, dout);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && n > 0) e = cudaMemcpy(out, dout, 2 * (size_t)n * sizeof(double), cudaMemcpyDeviceToHost);
  return cuda_check(nullptr, e, "coriolis_force");
}

int swf_dev_wind_force(int n, const double* in, double wx, double wy, const swf_params* P,
                       double* out) {
  Bufs B;
  double *din, *dout;
  swf_terrain T{1, 1, 1.0, 0.0, 0.0, nullptr};
  cudaError_t e = B.up(&din, in, 3 * (size_t)n);
  if (e == cudaSuccess) e = B.alloc(&dout, 2 * (size_t)n);
  if (e == cudaSuccess && n > 0) {
    k_wind<<<nblk(n), FT>>>(n, din, wx, wy, phys_of(&T, P), dout);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && n > 0) e = cudaMemcpy(out, dout, 2 * (size_t)n * sizeof(double), cudaMemcpyDeviceToHost);
  return cuda_check(nullptr, e, "wind_force");
}

int swf_dev_block_mask(int nx, int ny, const double* H, const uint8_t* index_q, double eps_dry,
                       int block_size, int* interior, int* halo) {
  if (nx <= 0 || ny <= 0) return set_err(nullptr, SWF_ECONFIG, "grid dimensions must be positive");
  if (block_size <= 0) return set_err(nullptr, SWF_ECONFIG, "block_size must be positive");
  const size_t n = (size_t)nx * ny;
  const int nbx = (nx + block_size - 1) / block_size, nby = (ny + block_size - 1) / block_size;
  const size_t nb = (size_t)nbx * nby;
  Bufs B;
  double* dH;
  unsigned char* dq = nullptr;
  int *di, *dh;
  cudaError_t e = B.up(&dH, H, n);
  if (e == cudaSuccess && index_q) e = B.up(&dq, (const unsigned char*)index_q, n);
  if (e == cudaSuccess) e = B.alloc(&di, nb);
  if (e == cudaSuccess) e = B.alloc(&dh, nb);
  if (e == cudaSuccess) {
    k_block_mask<<<nblk(nb), FT>>>(nx, ny, dH, dq, eps_dry, block_size, nbx, nby, di, dh);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(interior, di, nb * sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(halo, dh, nb * sizeof(int), cudaMemcpyDeviceToHost);
  return cuda_check(nullptr, e, "compute_block_mask");
}

int swf_dev_source_terms(const swf_terrain* T, const swf_source* S, int ns, double t,
                         int resample, double* sigma, double* vx, double* vy, uint8_t* index_q) {
  if (int rc = grid_ok(T)) return rc;
  // the geometry checks of SourceSpec::validate (sources.cpp:21-25) that keep
  // the fill in bounds; the C++ wrapper runs the full validate() first
  for (int m = 0; m < ns; ++m) {
    const swf_source& s = S[m];
    if (s.i0 > s.i1 || s.j0 > s.j1) return set_err(nullptr, SWF_ECONFIG, "empty cell rectangle");
    if (s.i0 < 0 || s.j0 < 0 || s.i1 >= T->nx || s.j1 >= T->ny)
      return set_err(nullptr, SWF_ECONFIG, "cells outside grid");
  }
  const size_t n = (size_t)T->nx * T->ny;
  std::vector<DevSrc> ds(ns > 0 ? ns : 1);
  std::vector<double> ht, hq;
  for (int m = 0; m < ns; ++m) {
    const swf_source& s = S[m];
    DevSrc& d = ds[m];
    d.kind = s.kind;
    d.i0 = s.i0;
    d.j0 = s.j0;
    d.i1 = s.i1;
    d.j1 = s.j1;
    d.nh = s.n_hydro;
    d.off = (int)ht.size();
    d.rate = s.rate;
    d.vx = s.vx;
    d.vy = s.vy;
    const int count = (s.i1 - s.i0 + 1) * (s.j1 - s.j0 + 1);
    d.count_area = count * (T->h * T->h);  // CellRect::count() * cell_area(), sources.cpp:40
    for (int q = 0; q < s.n_hydro; ++q) {
      ht.push_back(s.hydro_t[q]);
      hq.push_back(s.hydro_q[q]);
    }
  }
  Bufs B;
  DevSrc* dsrc;
  double *dht, *dhq, *dsig, *dS, *dX = nullptr, *dY = nullptr;
  unsigned char* dQ = nullptr;
  cudaError_t e = B.up(&dsrc, ds.data(), ds.size());
  if (e == cudaSuccess) e = B.up(&dht, ht.data(), ht.size());
  if (e == cudaSuccess) e = B.up(&dhq, hq.data(), hq.size());
  if (e == cudaSuccess) e = B.alloc(&dsig, ds.size());
  if (e == cudaSuccess) e = B.alloc(&dS, n);
  if (e == cudaSuccess && !resample) e = B.alloc(&dX, n);
  if (e == cudaSuccess && !resample) e = B.alloc(&dY, n);
  if (e == cudaSuccess && !resample) e = B.alloc(&dQ, n);
  if (e == cudaSuccess && ns > 0) {
    k_spec_sigma<<<nblk(ns), FT>>>(dsrc, ns, dht, dhq, t, dsig);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && !resample) e = cudaMemset(dX, 0, n * sizeof(double));
  if (e == cudaSuccess && !resample) e = cudaMemset(dY, 0, n * sizeof(double));
  if (e == cudaSuccess) {
    k_source_fill<<<nblk(n), FT>>>(T->nx, T->ny, dsrc, ns, dsig, resample, dS, dX, dY, dQ);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(sigma, dS, n * sizeof(double), cudaMemcpyDeviceToHost);
  if (!resample) {
    if (e == cudaSuccess) e = cudaMemcpy(vx, dX, n * sizeof(double), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(vy, dY, n * sizeof(double), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(index_q, dQ, n, cudaMemcpyDeviceToHost);
  }
  return cuda_check(nullptr, e, resample ? "resample_sigma" : "source_terms");
}

}  // extern "C"
