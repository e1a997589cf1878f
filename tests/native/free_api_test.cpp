// Every public declaration of the reference's step-path headers that the
// stepper test (dropin_test.cpp) does not reach: the free functions of
// forcing.hpp:29-57, block.hpp:38-52, sources.hpp:40-46, riemann.hpp:18-19,
// the stepper's copy/move semantics and its HalfView declaration.
//
// The SAME source is compiled two ways (tests/test_dropin_cpp.py):
//  * against the reference headers, linked with the reference objects that
//    oracle/Makefile compiles from /root/reference (in this container only):
//    its output is the committed fixture tests/golden/free_api_ref.bin
//    (tests/golden/make_free_golden.py);
//  * against this repository's include/ and libswflood_b200.so: on the GPU
//    its output must equal the fixture byte for byte.
// Test infrastructure.  Usage: free_api_test OUT.bin
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <exception>
#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <vector>

#include "swflood/block.hpp"
#include "swflood/forcing.hpp"
#include "swflood/grid.hpp"
#include "swflood/riemann.hpp"
#include "swflood/sources.hpp"
#include "swflood/stepper.hpp"

using namespace swflood;

static_assert(std::is_copy_constructible_v<CsphTvdStepper>, "stepper.hpp:76 is copyable");
static_assert(std::is_copy_assignable_v<CsphTvdStepper>, "stepper.hpp:76 is copy-assignable");
static_assert(std::is_move_constructible_v<CsphTvdStepper>, "stepper.hpp:76 is movable");
using HalfViewDeclared = CsphTvdStepper::HalfView;  // stepper.hpp:121

static FILE* out = nullptr;
static void put(double v) { std::fwrite(&v, sizeof v, 1, out); }
static void put(Vec2 v) {
  put(v.x);
  put(v.y);
}
static void put(const std::vector<double>& v) { std::fwrite(v.data(), sizeof(double), v.size(), out); }
static void put_i(long long v) { put((double)v); }
static void put(const std::vector<int>& v) {
  for (int x : v) put_i(x);
}
static void put(const std::vector<std::uint8_t>& v) {
  for (auto x : v) put_i(x);
}
static void put(const ForceField& f) {
  put_i(f.nx);
  put_i(f.ny);
  put(f.fx);
  put(f.fy);
  put(f.fric_x);
  put(f.fric_y);
  put(f.sigma_eff);
}
static void put(const SourceField& f) {
  put(f.sigma);
  put(f.vx);
  put(f.vy);
  put(f.index_q);
}
static void put(const BlockMask& m) {
  put_i(m.block_size);
  put_i(m.nbx);
  put_i(m.nby);
  put(m.interior_wet);
  put(m.halo_wet);
  put(active_fraction(m));
  for (StageKind k : {StageKind::Lagrangian, StageKind::Flux, StageKind::Final}) {
    std::vector<int> a = active_blocks(m, k);
    put_i((long long)a.size());
    put(a);
    long long sum_body = 0, sum_skip = 0, n_body = 0, n_skip = 0;
    for_each_active_block(
        m, k, [&](int ib) { sum_body += ib, ++n_body; }, [&](int ib) { sum_skip += ib, ++n_skip; });
    put_i(sum_body);
    put_i(n_body);
    put_i(sum_skip);
    put_i(n_skip);
    long long n_only = 0;
    for_each_active_block(m, k, [&](int) { ++n_only; });
    put_i(n_only);
  }
}

// seed 0: the fixed case of tests/golden/free_api_ref.bin.gz; seed > 0: the
// same program on a seeded random variant (grid shape, bed, water level,
// films, momenta, Manning field, viscosity, latitude, wind, sources), whose
// reference outputs are tests/golden/free_api_ref_s<seed>.bin.gz
static unsigned long long rng_state = 0;
static double U(double a, double b, double fixed) {
  if (!rng_state) return fixed;
  rng_state ^= rng_state << 13;
  rng_state ^= rng_state >> 7;
  rng_state ^= rng_state << 17;
  return a + (b - a) * (double)(rng_state >> 11) * (1.0 / 9007199254740992.0);
}
static int Ui(int a, int b, int fixed) {  // [a, b]
  return rng_state ? std::min(b, a + (int)U(0.0, (double)(b - a + 1), 0.0)) : fixed;
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  out = std::fopen(argv[1], "wb");
  if (!out) return 2;
  if (argc > 2) rng_state = 0x9E3779B97F4A7C15ull * (unsigned long long)std::atoll(argv[2]);

  // a tilted, bumpy basin: wet pools, dry banks above and below the water
  // surface, a thin film near eps_dry, a Manning field
  const int nx = Ui(5, 48, 41), ny = Ui(5, 40, 29);
  const double slope = U(-4e-3, 4e-3, 2e-3), amp = U(0.1, 2.0, 0.9), kx = U(0.05, 0.8, 0.31),
               ky = U(0.05, 0.8, 0.23), level = U(-0.5, 1.2, 0.6);
  const int film_a = Ui(5, 40, 23), film_b = Ui(5, 40, 31);
  Terrain T;
  T.nx = nx;
  T.ny = ny;
  T.h = U(0.5, 60.0, 12.5);
  T.b.resize(T.cells());
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i)
      T.b[T.idx(i, j)] = slope * T.xc(i) + amp * std::cos(kx * i) * std::sin(ky * j + 0.4);
  PhysicalParams P;
  P.nu = U(0.0, 3.0, 0.75);
  P.omega_z = latitude_to_omega_z(U(-80.0, 80.0, 48.7));
  P.n_field.resize(T.cells());
  for (int k = 0; k < (int)T.cells(); ++k) P.n_field[k] = 0.02 + 0.015 * ((k * 7) % 5) / 4.0;
  const double vx = U(-1.5, 1.5, 0.3), vy = U(-1.5, 1.5, 0.25);
  FlowState S = FlowState::dry(T);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int k = S.idx(i, j);
      double e = level + 0.25 * std::sin(0.17 * i + 0.05 * j);
      S.H[k] = std::max(0.0, e - T.b[k]);
      if ((i * 13 + j * 7) % film_a == 0) S.H[k] = 0.6e-6;  // just above eps_dry
      if ((i * 5 + j * 11) % film_b == 0) S.H[k] = 0.4e-6;  // dry film
      S.HUx[k] = S.H[k] * (vx * std::cos(0.2 * j) - 0.1);
      S.HUy[k] = S.H[k] * (vy * std::sin(0.3 * i));
    }
  S.enforce_dry_rule(P.eps_dry);
  WindForcing W;
  W.series = {{0.0, U(-20, 20, 4.0), U(-20, 20, -1.0)},
              {100.0, U(-20, 20, 6.5), U(-20, 20, 2.0)},
              {250.0, U(-20, 20, -3.0), U(-20, 20, 5.0)}};
  WindForcing none;

  auto rect = [&](int i0, int j0, int i1, int j1) {
    CellRect c;
    c.i0 = Ui(0, nx - 1, i0);
    c.j0 = Ui(0, ny - 1, j0);
    c.i1 = Ui(c.i0, nx - 1, i1);
    c.j1 = Ui(c.j0, ny - 1, j1);
    return c;
  };
  std::vector<SourceSpec> src(3);
  src[0].kind = SourceSpec::Kind::Discharge;
  src[0].name = "inflow";
  src[0].cells = rect(0, 10, 2, 15);
  src[0].hydrograph = {{0.0, U(0, 500, 10.0)}, {60.0, U(0, 500, 250.0)}, {300.0, U(0, 500, 40.0)}};
  src[0].source_velocity = {U(-1, 1, 0.8), U(-1, 1, -0.1)};
  src[1].kind = SourceSpec::Kind::Rain;
  src[1].name = "rain";
  src[1].cells = rect(1, 12, 30, 20);  // overlaps the inflow
  src[1].rate = U(0.0, 1e-3, 2.5e-5);
  src[2].kind = SourceSpec::Kind::Discharge;
  src[2].name = "drain";
  src[2].cells = rect(38, 3, 40, 6);
  src[2].hydrograph = {{0.0, U(-100, 0, -15.0)}};
  src[2].source_velocity = {U(-1, 1, -0.2), U(-1, 1, 0.3)};

  // forcing.hpp:34-47 at every cell
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      put(viscous_force(S, P, T, i, j));
      put(surface_gradient_force(S, T, P, i, j));
    }
  // forcing.hpp:29-43, riemann.hpp:18-19 on sampled states
  for (int q = 0; q < 64; ++q) {
    Vec2 u{0.37 * std::sin(0.7 * q) - 0.05, 0.29 * std::cos(1.3 * q)};
    double H = 1e-5 + 0.11 * q;
    put(coriolis_force(u, P));
    put(wind_force(u, H, W, 3.7 * q + 0.5, P));
    put(bottom_friction(u, H, P));
    put(bottom_friction(u, H, 9.81, 0.013 + 0.001 * q));
    FaceFlux f = hll_face_flux(H, u.x, u.y, q % 3 == 0 ? 0.0 : 0.5 * H + 0.01, -u.y, u.x, P.g);
    put(f.fm);
    put(f.fn);
    put(f.ft);
  }
  // sources.hpp:40-46
  for (double t : {0.0, 37.5, 60.0, 145.25, 400.0}) {
    SourceField F = source_terms(src, t, T);
    put(F);
    SourceField G = F;
    resample_sigma(src, t + 13.0, T, G);
    put(G);
  }
  // forcing.hpp:51-54 with and without sources / wind, both Manning forms
  SourceField F = source_terms(src, 80.0, T);
  SourceField empty;
  put(assemble_forces(S, T, P, W, F, 80.0));
  put(assemble_forces(S, T, P, none, empty, 0.0));
  PhysicalParams Pn = P;
  Pn.n_field.clear();
  Pn.n_manning = 0.031;
  Pn.nu = 0.0;
  put(assemble_forces(S, T, Pn, W, empty, 205.0));
  // block.hpp:38-52
  for (int bs : {1, 4, 7, 16, 64}) {
    put(compute_block_mask(S, F, P.eps_dry, bs));
    put(compute_block_mask(S, empty, P.eps_dry, bs));
  }

  // stepper.hpp:76: copies step like the original
  TimestepControl K;
  StepperOptions O;
  O.block_size = 8;
  O.boundaries.east = EdgeKind::Open;
  CsphTvdStepper a(T, P, K, O);
  a.set_wind(W);
  a.set_sources(src);
  CsphTvdStepper b(a);             // copy after configuration
  CsphTvdStepper c(T, Pn, K, {});  // replaced by copy assignment below
  c = a;
  CsphTvdStepper d(std::move(c));
  FlowState Sa = S, Sb = S, Sd = S;
  try {  // (a random variant may abort: the message is part of the output)
    for (int n = 0; n < 6; ++n) {
      StepInfo ia = a.step(Sa), ib = b.step(Sb), id = d.step(Sd);
      put(ia.tau);
      put(ib.tau);
      put(id.tau);
      put_i(ia.flux_blocks);
      put_i(id.lagrangian_blocks);
    }
  } catch (const std::exception& e) {
    put_i(-1);
    const std::string m = e.what();
    std::fwrite(m.data(), 1, m.size(), out);
  }
  put(Sa.t);
  put(Sa.H);
  put(Sa.HUx);
  put(Sa.HUy);
  put(Sb.H);
  put(Sb.HUx);
  put(Sb.HUy);
  put(Sd.H);
  put(Sd.HUx);
  put(Sd.HUy);
  put(d.mask().interior_wet);
  std::fclose(out);
  std::printf("free_api ok\n");
  return 0;
}
