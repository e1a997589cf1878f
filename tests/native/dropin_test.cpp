// A program written against the REFERENCE's C++ API (swflood::CsphTvdStepper,
// proj/include/swflood/stepper.hpp), built against this repository's drop-in
// headers and linked with libswflood_b200.so.  It checks the GPU results
// against the C restatement of the reference (oracle/liborc.so, linked as the
// checker) bit for bit and exercises the stage interface and accessors.
// Test infrastructure: built and run by tests/test_dropin_cpp.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "swflood/stepper.hpp"
#include "../../oracle/swf_oracle.h"

using namespace swflood;

static int fails = 0;
#define CHECK(c, ...)                      \
  do {                                     \
    if (!(c)) {                            \
      std::printf("FAIL: " __VA_ARGS__);   \
      std::printf("\n");                   \
      ++fails;                             \
    }                                      \
  } while (0)

static bool same_bits(const std::vector<double>& a, const double* b) {
  return std::memcmp(a.data(), b, a.size() * sizeof(double)) == 0;
}

int main() {
  // a sloped, bumpy basin with a drain, rain, wind, Coriolis and viscosity
  const int nx = 96, ny = 80;
  Terrain T;
  T.nx = nx;
  T.ny = ny;
  T.h = 25.0;
  T.b.resize(T.cells());
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i)
      T.b[T.idx(i, j)] = 1e-3 * T.xc(i) + 0.7 * std::cos(0.11 * i) * std::sin(0.07 * j);
  PhysicalParams P;
  P.nu = 0.5;
  P.omega_z = latitude_to_omega_z(48.7);
  TimestepControl K;
  StepperOptions O;
  O.boundaries.east = EdgeKind::Open;
  FlowState S = FlowState::dry(T);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx / 3; ++i) S.H[S.idx(i, j)] = std::max(0.0, 2.5 - T.b[T.idx(i, j)]);
  std::vector<SourceSpec> src(2);
  src[0].name = "drain";
  src[0].cells = {70, 30, 72, 33};
  src[0].hydrograph = {{0.0, -5.0}, {50.0, -20.0}};
  src[1].kind = SourceSpec::Kind::Rain;
  src[1].name = "rain";
  src[1].cells = {10, 50, 40, 70};
  src[1].rate = 2e-5;
  WindForcing W = WindForcing::constant(4.0, -1.0);

  CsphTvdStepper gpu(T, P, K, O);
  gpu.set_wind(W);
  gpu.set_sources(src);

  // the checker through its C ABI
  swf_terrain ct{nx, ny, T.h, 0.0, 0.0, T.b.data()};
  swf_params cp{P.g, P.n_manning, P.nu, P.omega_z, P.c_a, P.rho_air, P.rho_water, P.eps_dry, nullptr};
  swf_control ck{K.courant, K.dt_max, K.dt_min};
  swf_options co{16, 1, 1, SWF_EDGE_REFLECTIVE, SWF_EDGE_OPEN, SWF_EDGE_REFLECTIVE, SWF_EDGE_REFLECTIVE};
  orc_ctx* orc = nullptr;
  CHECK(orc_create(&ct, &cp, &ck, &co, &orc) == 0, "orc_create");
  double wt = 0.0, wx = 4.0, wy = -1.0;
  orc_set_wind(orc, 1, &wt, &wx, &wy);
  double ht[2] = {0.0, 50.0}, hq[2] = {-5.0, -20.0};
  swf_source cs[2] = {{SWF_SOURCE_DISCHARGE, 70, 30, 72, 33, 2, ht, hq, 0.0, 0.0, 0.0},
                      {SWF_SOURCE_RAIN, 10, 50, 40, 70, 0, nullptr, nullptr, 2e-5, 0.0, 0.0}};
  orc_set_sources(orc, 2, cs);
  orc_set_state(orc, S.H.data(), S.HUx.data(), S.HUy.data(), S.t);

  std::vector<double> H(T.cells()), X(T.cells()), Y(T.cells());
  for (int n = 0; n < 40; ++n) {
    StepInfo a = gpu.step(S);
    swf_step_info b;
    orc_step(orc, 0.0, &b);
    CHECK(a.tau == b.tau, "tau step %d", n);
    CHECK(a.flux_blocks == b.flux_blocks, "flux blocks step %d", n);
  }
  double t;
  orc_get_state(orc, H.data(), X.data(), Y.data(), &t);
  CHECK(same_bits(S.H, H.data()) && same_bits(S.HUx, X.data()) && same_bits(S.HUy, Y.data()),
        "state after 40 steps");
  CHECK(S.t == t, "time");

  // stage interface + accessors (stepper.hpp:88-119)
  gpu.begin_step(S);
  gpu.compute_forces(S);
  double tau = gpu.compute_dt(S);
  gpu.predictor(S, tau);
  gpu.mid_forces(S, tau);
  gpu.corrector(S, tau);
  gpu.flux(S, tau);
  orc_stage(orc, SWF_STAGE_BEGIN, 0, nullptr);
  orc_stage(orc, SWF_STAGE_FORCES, 0, nullptr);
  double tau2 = 0;
  orc_stage(orc, SWF_STAGE_DT, 0.0, &tau2);
  CHECK(tau == tau2, "stage tau");
  for (int s = SWF_STAGE_PREDICTOR; s <= SWF_STAGE_FLUX; ++s) orc_stage(orc, s, tau2, nullptr);
  orc_scratch(orc, SWF_SCR_FH, H.data());
  auto fh = gpu.flux_mass();
  CHECK(std::memcmp(fh.data(), H.data(), fh.size() * sizeof(double)) == 0, "flux_mass");
  orc_scratch(orc, SWF_SCR_FM_FX, H.data());
  CHECK(same_bits(gpu.forces_mid().fx, H.data()), "forces_mid().fx");
  orc_scratch(orc, SWF_SCR_DRX, H.data());
  auto dx = gpu.displacement_x();
  CHECK(std::memcmp(dx.data(), H.data(), dx.size() * sizeof(double)) == 0, "displacement_x");
  const BlockMask& m = gpu.mask();
  CHECK(m.total_blocks() == 6 * 5, "mask blocks %d", m.total_blocks());
  gpu.final_update(S, tau);
  orc_stage(orc, SWF_STAGE_FINAL, tau2, nullptr);
  orc_get_state(orc, H.data(), X.data(), Y.data(), &t);
  CHECK(same_bits(S.H, H.data()) && same_bits(S.HUx, X.data()), "state after stage step");

  // errors: ConfigError with the reference's message
  try {
    TimestepControl bad;
    bad.courant = 2.0;
    CsphTvdStepper x(T, P, bad, O);
    CHECK(false, "no ConfigError");
  } catch (const ConfigError& e) {
    CHECK(std::strstr(e.what(), "Courant") != nullptr, "message");
  }
  // free functions on the device
  Vec2 f = bottom_friction({1.0, 0.0}, 1.0, 9.81, 0.02);
  CHECK(std::fabs(f.x + 3.924e-3) < 1e-15 && f.y == 0.0, "friction KAT");
  FaceFlux ff = hll_face_flux(2.0, 0.0, 0.0, 2.0, 0.0, 0.0, 9.81);
  CHECK(ff.fm == 0.0 && std::fabs(ff.fn - 19.62) < 1e-12, "hll equal states");
  orc_destroy(orc);
  std::printf("%s (%d failures)\n", fails ? "FAILED" : "dropin ok", fails);
  return fails ? 1 : 0;
}
