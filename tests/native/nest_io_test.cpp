// C++ users of the SPEC-only modules (include/swflood/nesting.hpp, io.hpp):
// ESRI ASCII round trip, a scenario file, and a two-level nested run whose
// volume ledger balances (flux-corrected coupling).
// Test infrastructure: built and run by tests/test_dropin_cpp.py.
#include <cmath>
#include <cstdio>
#include <string>

#include "swflood/io.hpp"
#include "swflood/nesting.hpp"

using namespace swflood;

static int fails = 0;
#define CHECK(c, ...)                    \
  do {                                   \
    if (!(c)) {                          \
      std::printf("FAIL: " __VA_ARGS__); \
      std::printf("\n");                 \
      ++fails;                           \
    }                                    \
  } while (0)

int main(int argc, char** argv) {
  std::string dir = argc > 1 ? argv[1] : "/tmp";
  // ---- ESRI ASCII: write a bed, read it back (rows north -> south) ------------
  const int n = 96, r = 4, i0 = 36, j0 = 32, ni = 24, nj = 28, gw = 2;
  const double h = 20.0;
  Terrain T;
  T.nx = T.ny = n;
  T.h = h;
  T.b.resize(T.cells());
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      T.b[T.idx(i, j)] = 0.02 * (n - i) + 0.5 * std::sin(0.21 * i) * std::cos(0.17 * j);
  io::write_raster(dir + "/bed.asc", n, n, 0.0, 0.0, h, T.b, -9999.0, 17);
  Terrain R = io::load_terrain(dir + "/bed.asc");
  CHECK(R.nx == n && R.ny == n && R.h == h, "raster header");
  bool same = true;
  for (size_t k = 0; k < T.b.size(); ++k) same = same && R.b[k] == T.b[k];
  CHECK(same, "raster values (%%.17e round trip)");
  bool threw = false;
  try {
    io::load_terrain(dir + "/missing.asc");
  } catch (const ConfigError&) {
    threw = true;
  }
  CHECK(threw, "missing raster is a ConfigError");

  // ---- nested run: the global bed over the window = block mean of the fine bed
  NestWindow w{i0, j0, ni, nj, r, gw, true};
  Terrain F;
  F.nx = w.fine_nx();
  F.ny = w.fine_ny();
  F.h = h / r;
  F.x0 = i0 * h - gw * F.h;
  F.y0 = j0 * h - gw * F.h;
  F.b.resize(F.cells());
  for (int j = 0; j < F.ny; ++j)
    for (int i = 0; i < F.nx; ++i) {
      double x = F.x0 + (i + 0.5) * F.h, y = F.y0 + (j + 0.5) * F.h;
      double xi = x / h - 0.5, yj = y / h - 0.5;
      F.b[F.idx(i, j)] = 0.02 * (n - xi) + 0.5 * std::sin(0.21 * xi) * std::cos(0.17 * yj);
    }
  for (int cj = 0; cj < nj; ++cj)
    for (int ci = 0; ci < ni; ++ci) {
      double s = 0.0;
      for (int b = 0; b < r; ++b)
        for (int a = 0; a < r; ++a) s += F.b[F.idx(gw + ci * r + a, gw + cj * r + b)];
      R.b[R.idx(i0 + ci, j0 + cj)] = s / (r * r);
    }
  PhysicalParams P;
  P.n_manning = 0.03;
  CsphTvdStepper global(R, P, TimestepControl{});
  NestedGrid zoom(global, w, F, P);
  CHECK(zoom.bathymetry_deviation() < 1e-12, "consistent beds: %g", zoom.bathymetry_deviation());
  // a wave from the west over a partly wet valley
  FlowState G = FlowState::dry(R), S = FlowState::dry(F);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      double d = (i < 20 ? 2.6 : 1.6) - R.b[R.idx(i, j)];
      G.H[G.idx(i, j)] = d > 1e-6 ? d : 0.0;
    }
  for (int j = 0; j < F.ny; ++j)
    for (int i = 0; i < F.nx; ++i) {
      double d = 1.6 - F.b[F.idx(i, j)];
      S.H[S.idx(i, j)] = d > 1e-6 ? d : 0.0;
    }
  zoom.set_state(S);
  // coarse window cells = fine means (consistent start)
  {
    FlowState f = zoom.state();
    for (int cj = 0; cj < nj; ++cj)
      for (int ci = 0; ci < ni; ++ci) {
        double s = 0.0;
        for (int b = 0; b < r; ++b)
          for (int a = 0; a < r; ++a) s += f.H[f.idx(gw + ci * r + a, gw + cj * r + b)];
        G.H[G.idx(i0 + ci, j0 + cj)] = s / (r * r);
      }
  }
  double v0 = total_volume(G, R), ledger = 0.0;
  int subs = 0;
  for (int k = 0; k < 40; ++k) {
    CoupledStepInfo ci = coupled_step(global, G, {&zoom});
    ledger += ci.reflux_clamp_volume + ci.global.clamp_deficit_volume;
    subs += ci.substeps_total;
  }
  double v1 = total_volume(G, R);
  CHECK(subs >= 40, "fine subcycling (%d substeps)", subs);
  CHECK(std::fabs((v1 - v0) - ledger) <= 1e-11 * v0, "ledger: dV=%g logged=%g", v1 - v0, ledger);
  FlowState fz = zoom.state();
  CHECK(fz.t == G.t, "levels synchronised (%g vs %g)", fz.t, G.t);
  io::write_snapshot(G, R, P, dir, "nest");
  Terrain eta = io::load_terrain(dir + "/nest_eta.asc");
  CHECK(eta.nx == n, "snapshot raster");
  std::printf(fails ? "nest_io FAILED (%d)\n" : "nest_io ok: %d substeps, dV %.3e, ledger %.3e\n",
              fails ? fails : subs, v1 - v0, ledger);
  return fails ? 1 : 0;
}
