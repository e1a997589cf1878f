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

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  out = std::fopen(argv[1], "wb");
  if (!out) return 2;

  // a tilted, bumpy basin: wet pools, dry banks above and below the water
  // surface, a thin film near eps_dry, a Manning field
  const int nx = 41, ny = 29;
  Terrain T;
  T.nx = nx;
  T.ny = ny;
  T.h = 12.5;
  T.b.resize(T.cells());
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i)
      T.b[T.idx(i, j)] = 2e-3 * T.xc(i) + 0.9 * std::cos(0.31 * i) * std::sin(0.23 * j + 0.4);
  PhysicalParams P;
  P.nu = 0.75;
  P.omega_z = latitude_to_omega_z(48.7);
  P.n_field.resize(T.cells());
  for (int k = 0; k < (int)T.cells(); ++k) P.n_field[k] = 0.02 + 0.015 * ((k * 7) % 5) / 4.0;
  FlowState S = FlowState::dry(T);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int k = S.idx(i, j);
      double e = 0.6 + 0.25 * std::sin(0.17 * i + 0.05 * j);
      S.H[k] = std::max(0.0, e - T.b[k]);
      if ((i * 13 + j * 7) % 23 == 0) S.H[k] = 0.6e-6;  // just above eps_dry
      if ((i * 5 + j * 11) % 31 == 0) S.H[k] = 0.4e-6;  // dry film
      S.HUx[k] = S.H[k] * (0.3 * std::cos(0.2 * j) - 0.1);
      S.HUy[k] = S.H[k] * (0.25 * std::sin(0.3 * i));
    }
  S.enforce_dry_rule(P.eps_dry);
  WindForcing W;
  W.series = {{0.0, 4.0, -1.0}, {100.0, 6.5, 2.0}, {250.0, -3.0, 5.0}};
  WindForcing none;

  std::vector<SourceSpec> src(3);
  src[0].kind = SourceSpec::Kind::Discharge;
  src[0].name = "inflow";
  src[0].cells = {0, 10, 2, 15};
  src[0].hydrograph = {{0.0, 10.0}, {60.0, 250.0}, {300.0, 40.0}};
  src[0].source_velocity = {0.8, -0.1};
  src[1].kind = SourceSpec::Kind::Rain;
  src[1].name = "rain";
  src[1].cells = {1, 12, 30, 20};  // overlaps the inflow
  src[1].rate = 2.5e-5;
  src[2].kind = SourceSpec::Kind::Discharge;
  src[2].name = "drain";
  src[2].cells = {38, 3, 40, 6};
  src[2].hydrograph = {{0.0, -15.0}};
  src[2].source_velocity = {-0.2, 0.3};

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
  for (int n = 0; n < 6; ++n) {
    StepInfo ia = a.step(Sa), ib = b.step(Sb), id = d.step(Sd);
    put(ia.tau);
    put(ib.tau);
    put(id.tau);
    put_i(ia.flux_blocks);
    put_i(id.lagrangian_blocks);
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
