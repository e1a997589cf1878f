// swflood — command-line driver of the B200 step (SPEC.md [MODULE]
// scenario_io cli_run, and [MODULE] validation run_case,
// SPEC.md:513-521).  The reference ships no CLI ("callers");
// this one drives the drop-in C++ API (libswflood_b200.so) and the resident
// C ABI of libswflood_cuda.so.
//
//   swflood run <scenario> [--out DIR] [--no-skip] [--block-size B] [--workers N]
//   swflood bench <scenario> [--steps K]
//   swflood info <terrain.asc>
//   swflood validate <case> [--resolution N] [--seed S] [--out DIR]
//
// Exit codes: 0 success, 1 configuration error / usage, 2 numerical abort.
#include <sys/stat.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "swflood/io.hpp"
#include "swflood/nesting.hpp"
#include "swflood_b200.hpp"

using namespace swflood;

namespace {

struct Args {
  std::string cmd, target, out = "swflood_out";
  bool no_skip = false;
  int block_size = 0, workers = 0, steps = 50, resolution = 0;
  unsigned seed = 1705;
};

const char* kUsage =
    "usage: swflood run <scenario> [--out DIR] [--no-skip] [--block-size B] [--workers N]\n"
    "       swflood bench <scenario> [--steps K] [--no-skip] [--block-size B]\n"
    "       swflood info <terrain.asc>\n"
    "       swflood validate <case> [--resolution N] [--seed S]\n"
    "cases: lake-at-rest dam-break skip-equivalence mass-ledger mirror-symmetry zoom-mass\n"
    "       speedup stage-shares all\n";

[[noreturn]] void usage(const std::string& why) {
  std::fprintf(stderr, "swflood: %s\n%s", why.c_str(), kUsage);
  throw ConfigError(why);
}

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 3) usage("missing subcommand or argument");
  a.cmd = argv[1];
  a.target = argv[2];
  for (int k = 3; k < argc; ++k) {
    std::string f = argv[k];
    auto val = [&]() -> std::string {
      if (k + 1 >= argc) usage("flag " + f + " needs a value");
      return argv[++k];
    };
    auto ival = [&]() {
      std::string v = val();
      char* e = nullptr;
      long x = std::strtol(v.c_str(), &e, 10);
      if (*e || v.empty()) usage("flag " + f + " needs an integer, got '" + v + "'");
      return (int)x;
    };
    if (f == "--out") a.out = val();
    else if (f == "--no-skip") a.no_skip = true;
    else if (f == "--block-size") a.block_size = ival();
    else if (f == "--workers") a.workers = ival();
    else if (f == "--steps") a.steps = ival();
    else if (f == "--resolution") a.resolution = ival();
    else if (f == "--seed") a.seed = (unsigned)ival();
    else usage("unknown flag " + f);
  }
  if (a.cmd != "run" && a.cmd != "bench" && a.cmd != "info" && a.cmd != "validate")
    usage("unknown subcommand '" + a.cmd + "'");
  return a;
}

void mkdirs(const std::string& d) {
  std::string acc;
  for (size_t i = 0; i <= d.size(); ++i) {
    if (i == d.size() || d[i] == '/') {
      if (!acc.empty()) mkdir(acc.c_str(), 0755);
    }
    if (i < d.size()) acc += d[i];
  }
}

void apply_flags(const Args& a, io::ScenarioConfig& c) {
  if (a.no_skip) c.options.skip_dry_blocks = false;
  if (a.block_size) c.options.block_size = a.block_size;
  if (a.workers) c.options.workers = a.workers;
}

void check(int rc, swf_ctx* c) {
  if (!rc) return;
  std::string m = swf_last_error(c);
  if (rc == SWF_ENUMERICAL) throw NumericalError(m);
  if (rc == SWF_ECONFIG) throw ConfigError(m);
  throw std::runtime_error(m);
}

// ---------------------------------------------------------------- run
int cmd_run(const Args& a) {
  io::ScenarioConfig cfg = io::load_scenario(a.target);
  apply_flags(a, cfg);
  Terrain T = io::scenario_terrain(cfg);
  FlowState s = io::scenario_initial_state(cfg, T);
  CsphTvdStepper st(T, cfg.params, cfg.control, cfg.options);
  if (cfg.wind.any()) st.set_wind(cfg.wind);
  if (!cfg.sources.empty()) st.set_sources(cfg.sources);
  mkdirs(a.out);
  io::SummaryWriter sum(a.out + "/summary.csv");
  swf_ctx* c = st.native();
  check(swf_upload_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), s.t), c);
  io::SummaryRow ledger;
  auto snapshot = [&](int idx, double tau) {
    check(swf_download_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), &s.t), c);
    io::SummaryRow r = io::summarize(s, T, cfg.params);
    r.tau = tau;
    r.steps = ledger.steps;
    r.source_volume = ledger.source_volume;
    r.outflow_volume = ledger.outflow_volume;
    r.clamp_deficit = ledger.clamp_deficit;
    sum.row(r);
    char stem[32];
    std::snprintf(stem, sizeof stem, "snap%05d", idx);
    io::write_snapshot(s, T, cfg.params, a.out, stem);
  };
  double t0 = s.t;
  int nsnap = (int)std::floor(cfg.duration / cfg.cadence + 1e-9);
  snapshot(0, 0.0);
  auto w0 = std::chrono::steady_clock::now();
  double t = t0, last_tau = 0.0;
  for (int k = 1; k <= nsnap; ++k) {
    double target = t0 + k * cfg.cadence;
    while (target - t > 1e-9 * cfg.cadence) {
      swf_step_info info;
      check(swf_step(c, target - t, &info), c);
      t += info.tau;
      last_tau = info.tau;
      ledger.steps++;
      ledger.source_volume += info.source_volume;
      ledger.outflow_volume += info.boundary_outflow_volume;
      ledger.clamp_deficit += info.clamp_deficit_volume;
    }
    snapshot(k, last_tau);
  }
  double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
  std::printf("run: %ld steps to t=%.6g s in %.3f s wall (%.1f Mcell-updates/s), %d snapshots in %s\n",
              ledger.steps, t, wall, T.cells() * (double)ledger.steps / wall / 1e6, sum.rows(),
              a.out.c_str());
  return 0;
}

// ---------------------------------------------------------------- info
int cmd_info(const Args& a) {
  Terrain T = io::load_terrain(a.target);
  double mn = *std::min_element(T.b.begin(), T.b.end());
  double mx = *std::max_element(T.b.begin(), T.b.end());
  double mean = 0.0;
  size_t nodata = 0;
  for (double v : T.b) {
    mean += v;
    nodata += v == io::kNoDataBed;
  }
  mean /= (double)T.b.size();
  std::printf("terrain %s: %d x %d cells, h = %g m, origin (%g, %g), extent %g x %g m\n",
              a.target.c_str(), T.nx, T.ny, T.h, T.x0, T.y0, T.nx * T.h, T.ny * T.h);
  std::printf("bed: min %.6g m, max %.6g m, mean %.6g m, NODATA cells %zu\n", mn, mx, mean, nodata);
  std::printf("device memory for a fused stepper: %.3f GB\n", T.cells() * 80.0 / 1e9);
  return 0;
}

// ---------------------------------------------------------------- bench
double time_steps(CsphTvdStepper& st, const FlowState& s0, int K, std::vector<double>* shares) {
  swf_ctx* c = st.native();
  check(swf_upload_state(c, s0.H.data(), s0.HUx.data(), s0.HUy.data(), s0.t), c);
  int done = 0;
  swf_step_info last;
  check(swf_run(c, 3, 0.0, &done, &last), c);
  check(swf_set_timing(c, K), c);
  auto w0 = std::chrono::steady_clock::now();
  check(swf_run(c, K, 0.0, &done, &last), c);
  check(swf_sync(c), c);
  double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
  if (shares) {
    std::vector<double> tk((size_t)K * 8);
    check(swf_timing_read(c, K, tk.data()), c);
    shares->assign(8, 0.0);
    for (int k = 0; k < K; ++k)
      for (int b = 0; b < 8; ++b) (*shares)[b] += tk[(size_t)k * 8 + b];
  }
  check(swf_set_timing(c, 0), c);
  return el / K;
}

int cmd_bench(const Args& a) {
  io::ScenarioConfig cfg = io::load_scenario(a.target);
  apply_flags(a, cfg);
  Terrain T = io::scenario_terrain(cfg);
  FlowState s = io::scenario_initial_state(cfg, T);
  auto make = [&](bool skip) {
    StepperOptions o = cfg.options;
    o.skip_dry_blocks = skip;
    auto p = std::make_unique<CsphTvdStepper>(T, cfg.params, cfg.control, o);
    if (cfg.wind.any()) p->set_wind(cfg.wind);
    if (!cfg.sources.empty()) p->set_sources(cfg.sources);
    return p;
  };
  std::vector<double> sh;
  auto on = make(true);
  double t_on = time_steps(*on, s, a.steps, &sh);
  auto off = make(false);
  double t_off = time_steps(*off, s, a.steps, nullptr);
  double tot = 0.0;
  for (double v : sh) tot += v;
  const char* names[8] = {"mask+sources", "forces+cfl", "tau", "-", "-", "-", "lagrange+flux+final",
                          "diagnostics"};
  std::printf("bench %s: %d x %d cells, %d steps\n", a.target.c_str(), T.nx, T.ny, a.steps);
  std::printf("  skip on : %.4f ms/step  %.1f Mcell-updates/s\n", t_on * 1e3, T.cells() / t_on / 1e6);
  std::printf("  skip off: %.4f ms/step  %.1f Mcell-updates/s\n", t_off * 1e3, T.cells() / t_off / 1e6);
  std::printf("  speedup from dry-block skipping: %.3fx\n", t_off / t_on);
  std::printf("  stage shares (device time, skip on):\n");
  for (int b = 0; b < 8; ++b)
    if (names[b][0] != '-') std::printf("    %-22s %6.2f %%\n", names[b], tot > 0 ? 100.0 * sh[b] / tot : 0.0);
  return 0;
}

// ---------------------------------------------------------------- validate
struct Report {
  std::string name;
  std::vector<std::pair<std::string, double>> metrics;
  std::string threshold;
  bool pass = false;
};

Terrain bumpy(int n, double h, unsigned seed, double amp_scale = 1.0) {
  io::ScenarioConfig c;
  c.synthetic = "lake " + std::to_string(n) + " " + std::to_string(h);
  c.seed = seed;
  Terrain T = io::scenario_terrain(c);
  for (double& v : T.b) v *= amp_scale;
  return T;
}

Report v_lake(const Args& a) {
  int n = a.resolution ? a.resolution : 128;
  Terrain T = bumpy(n, 10.0, a.seed);
  FlowState s = FlowState::dry(T);
  for (size_t k = 0; k < s.H.size(); ++k) s.H[k] = std::max(0.0, 0.0 - T.b[k]);
  for (double& x : s.H)
    if (x <= 1e-6) x = 0.0;
  FlowState s0 = s;
  CsphTvdStepper st(T, PhysicalParams{}, TimestepControl{}, StepperOptions{});
  swf_ctx* c = st.native();
  check(swf_upload_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), 0.0), c);
  int done = 0;
  swf_step_info last;
  check(swf_run(c, 1000, 0.0, &done, &last), c);
  check(swf_download_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), &s.t), c);
  double umax = 0.0, dh = 0.0;
  for (size_t k = 0; k < s.H.size(); ++k) {
    dh = std::max(dh, std::fabs(s.H[k] - s0.H[k]));
    if (s.H[k] > 1e-6)
      umax = std::max(umax, std::hypot(s.HUx[k] / s.H[k], s.HUy[k] / s.H[k]));
  }
  return {"lake-at-rest", {{"resolution", n}, {"steps", 1000}, {"max|U| m/s", umax}, {"max|dH| m", dh}},
          "max|U| <= 1e-10 and max|dH| <= 1e-12 (SPEC.md:540)", umax <= 1e-10 && dh <= 1e-12};
}

double ritter_H(double x, double t, double hl, double g) {
  double c0 = std::sqrt(g * hl);
  if (x <= -c0 * t) return hl;
  if (x >= 2.0 * c0 * t) return 0.0;
  double q = 2.0 * c0 - x / t;
  return q * q / (9.0 * g);
}

double dam_l1(int N, double t_end) {
  int ny = 4;
  double L = 200.0, h = L / N;
  Terrain T;
  T.nx = N;
  T.ny = ny;
  T.h = h;
  T.x0 = -L / 2;
  T.b.assign((size_t)N * ny, 0.0);
  FlowState s = FlowState::dry(T);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < N / 2; ++i) s.H[T.idx(i, j)] = 1.0;
  PhysicalParams P;
  P.n_manning = 0.0;
  CsphTvdStepper st(T, P, TimestepControl{}, StepperOptions{});
  swf_ctx* c = st.native();
  check(swf_upload_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), 0.0), c);
  double t = 0.0;
  while (t_end - t > 1e-12) {
    swf_step_info info;
    check(swf_step(c, t_end - t, &info), c);
    t += info.tau;
  }
  check(swf_download_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), &s.t), c);
  double e = 0.0;
  for (int i = 0; i < N; ++i) e += std::fabs(s.H[T.idx(i, 1)] - ritter_H(T.xc(i), s.t, 1.0, P.g)) * h;
  return e / L;
}

Report v_dam(const Args& a) {
  int n = a.resolution ? a.resolution : 200;
  double e1 = dam_l1(n, 10.0), e2 = dam_l1(2 * n, 10.0);
  return {"dam-break", {{"N", n}, {"L1(H) N", e1}, {"L1(H) 2N", e2}, {"ratio", e1 / e2}},
          "L1 error ratio N->2N >= 1.7 vs the Ritter solution at t=10 s (SPEC.md:542)", e1 / e2 >= 1.7};
}

FlowState partial_flood(const Terrain& T, double level) {
  FlowState s = FlowState::dry(T);
  for (size_t k = 0; k < s.H.size(); ++k) {
    double d = level - T.b[k];
    s.H[k] = d > 1e-6 ? d : 0.0;
  }
  return s;
}

Report v_skip(const Args& a) {
  int n = a.resolution ? a.resolution : 256;
  Terrain T = bumpy(n, 10.0, a.seed);
  FlowState s0 = partial_flood(T, -1.5);
  std::vector<FlowState> res;
  for (bool skip : {true, false}) {
    StepperOptions o;
    o.skip_dry_blocks = skip;
    CsphTvdStepper st(T, PhysicalParams{}, TimestepControl{}, o);
    FlowState s = s0;
    swf_ctx* c = st.native();
    check(swf_upload_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), 0.0), c);
    int done;
    swf_step_info last;
    check(swf_run(c, 50, 0.0, &done, &last), c);
    check(swf_download_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), &s.t), c);
    res.push_back(s);
  }
  bool same = std::memcmp(res[0].H.data(), res[1].H.data(), res[0].H.size() * 8) == 0 &&
              std::memcmp(res[0].HUx.data(), res[1].HUx.data(), res[0].H.size() * 8) == 0 &&
              std::memcmp(res[0].HUy.data(), res[1].HUy.data(), res[0].H.size() * 8) == 0 &&
              res[0].t == res[1].t;
  return {"skip-equivalence", {{"resolution", n}, {"steps", 50}, {"bitwise_equal", same ? 1.0 : 0.0}},
          "skip on vs off bitwise identical after 50 steps (SPEC.md:544)", same};
}

Report v_mass(const Args& a) {
  int n = a.resolution ? a.resolution : 256;
  Terrain T = bumpy(n, 10.0, a.seed);
  FlowState s = FlowState::dry(T);
  double L = n * T.h;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {  // tilted free surface: sloshing in a closed basin
      double d = (1.0 + 0.5 * (T.xc(i) / L - 0.5)) - T.b[T.idx(i, j)];
      s.H[T.idx(i, j)] = d > 1e-6 ? d : 0.0;
    }
  double v0 = total_volume(s, T);
  CsphTvdStepper st(T, PhysicalParams{}, TimestepControl{}, StepperOptions{});
  swf_ctx* c = st.native();
  check(swf_upload_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), 0.0), c);
  double deficit = 0.0;
  for (int k = 0; k < 2000; ++k) {
    swf_step_info info;
    check(swf_step(c, 0.0, &info), c);
    deficit += info.clamp_deficit_volume;
  }
  check(swf_download_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), &s.t), c);
  double drift = std::fabs(total_volume(s, T) - v0 - deficit) / v0;
  // with a single-cell 40 m/s-equivalent source (100000 m3/s over one 50 m cell)
  Terrain T2 = T;
  T2.h = 50.0;
  FlowState s2 = s;
  s2.t = 0.0;
  for (double& x : s2.HUx) x = 0.0;
  for (double& x : s2.HUy) x = 0.0;
  CsphTvdStepper st2(T2, PhysicalParams{}, TimestepControl{}, StepperOptions{});
  SourceSpec q;
  q.name = "gate";
  q.cells = {n / 2, n / 2, n / 2, n / 2};
  q.hydrograph = {{0.0, 100000.0}};
  st2.set_sources({q});
  swf_ctx* c2 = st2.native();
  double w0 = total_volume(s2, T2);
  check(swf_upload_state(c2, s2.H.data(), s2.HUx.data(), s2.HUy.data(), 0.0), c2);
  double src = 0.0, out = 0.0, def = 0.0;
  for (int k = 0; k < 200; ++k) {
    swf_step_info info;
    check(swf_step(c2, 0.0, &info), c2);
    src += info.source_volume;
    out += info.boundary_outflow_volume;
    def += info.clamp_deficit_volume;
  }
  check(swf_download_state(c2, s2.H.data(), s2.HUx.data(), s2.HUy.data(), &s2.t), c2);
  double w1 = total_volume(s2, T2);
  double ledger = std::fabs((w1 - w0) - (src - out + def)) / std::max(std::fabs(w1), 1e-300);
  return {"mass-ledger",
          {{"resolution", n}, {"closed-basin drift (2000 steps)", drift}, {"ledger residual (source, 200 steps)", ledger}},
          "drift <= 1e-11 and ledger <= 1e-10 relative (SPEC.md:541)", drift <= 1e-11 && ledger <= 1e-10};
}

Report v_mirror(const Args& a) {
  int n = a.resolution ? a.resolution : 128;
  Terrain T;
  T.nx = T.ny = n;
  T.h = 8.0;
  T.b.assign((size_t)n * n, 0.0);
  FlowState s = FlowState::dry(T);
  double c = n * T.h / 2.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i)
      if (std::hypot(T.xc(i) - c, T.yc(j) - c) < n * T.h / 6.0) s.H[T.idx(i, j)] = 2.0;
  CsphTvdStepper st(T, PhysicalParams{}, TimestepControl{}, StepperOptions{});
  swf_ctx* cx = st.native();
  check(swf_upload_state(cx, s.H.data(), s.HUx.data(), s.HUy.data(), 0.0), cx);
  int done;
  swf_step_info last;
  check(swf_run(cx, 200, 0.0, &done, &last), cx);
  check(swf_download_state(cx, s.H.data(), s.HUx.data(), s.HUy.data(), &s.t), cx);
  double asym = 0.0, hmax = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      asym = std::max(asym, std::fabs(s.H[T.idx(i, j)] - s.H[T.idx(n - 1 - i, j)]));
      asym = std::max(asym, std::fabs(s.H[T.idx(i, j)] - s.H[T.idx(i, n - 1 - j)]));
      hmax = std::max(hmax, s.H[T.idx(i, j)]);
    }
  return {"mirror-symmetry", {{"resolution", n}, {"steps", 200}, {"max mirror asymmetry of H (m)", asym}},
          "asymmetry <= 1e-12 * max H", asym <= 1e-12 * hmax};
}

Report v_zoom(const Args& a) {
  int n = a.resolution ? a.resolution : 128;
  Terrain T = bumpy(n, 50.0, a.seed);
  FlowState s = partial_flood(T, 0.0);
  CsphTvdStepper g(T, PhysicalParams{}, TimestepControl{}, StepperOptions{});
  NestWindow w{n / 2 - n / 8, n / 2 - n / 8, n / 4, n / 4, 4, 2, true};
  Terrain F;
  F.nx = w.fine_nx();
  F.ny = w.fine_ny();
  F.h = T.h / w.r;
  F.x0 = T.x0 + w.i0 * T.h - w.ghost * F.h;
  F.y0 = T.y0 + w.j0 * T.h - w.ghost * F.h;
  F.b.assign(F.cells(), 0.0);
  for (int j = 0; j < F.ny; ++j)  // piecewise-constant fine bed (consistent under restriction)
    for (int i = 0; i < F.nx; ++i) {
      int ci = w.i0 + (int)std::floor((i - w.ghost) / (double)w.r);
      int cj = w.j0 + (int)std::floor((j - w.ghost) / (double)w.r);
      F.b[F.idx(i, j)] = T.b[T.idx(ci, cj)];
    }
  NestedGrid nest(g, w, F, PhysicalParams{});
  FlowState fs = FlowState::dry(F);
  for (size_t k = 0; k < fs.H.size(); ++k) fs.H[k] = std::max(0.0, 0.0 - F.b[k]);
  nest.set_state(fs);
  double m0 = total_volume(s, T);
  check(swf_upload_state(g.native(), s.H.data(), s.HUx.data(), s.HUy.data(), 0.0), g.native());
  // a wave: raise the west third by 1 m
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n / 3; ++i) s.H[T.idx(i, j)] += 1.0;
  m0 = total_volume(s, T);
  check(swf_upload_state(g.native(), s.H.data(), s.HUx.data(), s.HUy.data(), 0.0), g.native());
  int subs = 0;
  double ledger = 0.0;
  for (int k = 0; k < 100; ++k) {
    CoupledStepInfo ci = coupled_step_resident(g, {&nest});
    subs += ci.substeps_total;
    ledger += ci.reflux_clamp_volume + ci.global.clamp_deficit_volume;
  }
  check(swf_download_state(g.native(), s.H.data(), s.HUx.data(), s.HUy.data(), &s.t), g.native());
  double dv = total_volume(s, T) - m0;
  double drift = std::fabs(dv - ledger) / m0;
  return {"zoom-mass",
          {{"resolution", n}, {"coupled steps", 100}, {"fine substeps", subs},
           {"relative volume change", dv / m0}, {"logged clamp volume / V0", ledger / m0},
           {"unaccounted drift", drift}},
          "unaccounted drift <= 1e-8 (SPEC.md:392; flux-corrected coupling)", drift <= 1e-8};
}

Report v_speedup(const Args& a) {
  int n = a.resolution ? a.resolution : 1024;
  Terrain T = bumpy(n, 50.0, a.seed);
  FlowState s = partial_flood(T, -2.0);
  double t[2];
  for (int k = 0; k < 2; ++k) {
    StepperOptions o;
    o.skip_dry_blocks = k == 0;
    CsphTvdStepper st(T, PhysicalParams{}, TimestepControl{}, o);
    t[k] = time_steps(st, s, 50, nullptr);
  }
  return {"speedup", {{"resolution", n}, {"ms/step skip", t[0] * 1e3}, {"ms/step no-skip", t[1] * 1e3}, {"speedup", t[1] / t[0]}},
          "skipping is faster on a partial flood", t[1] > t[0]};
}

Report v_shares(const Args& a) {
  int n = a.resolution ? a.resolution : 1024;
  Terrain T = bumpy(n, 50.0, a.seed);
  FlowState s = partial_flood(T, 0.0);
  CsphTvdStepper st(T, PhysicalParams{}, TimestepControl{}, StepperOptions{});
  std::vector<double> sh;
  time_steps(st, s, 50, &sh);
  double tot = 0.0;
  for (double v : sh) tot += v;
  return {"stage-shares",
          {{"forces+cfl %", 100 * sh[1] / tot}, {"lagrange+flux+final %", 100 * sh[6] / tot},
           {"other %", 100 * (tot - sh[1] - sh[6]) / tot}},
          "reported (paper Fig. 5: flux stage dominates)", sh[6] > sh[1]};
}

int cmd_validate(const Args& a) {
  std::map<std::string, std::function<Report(const Args&)>> cases = {
      {"lake-at-rest", v_lake},  {"dam-break", v_dam},       {"skip-equivalence", v_skip},
      {"mass-ledger", v_mass},   {"mirror-symmetry", v_mirror}, {"zoom-mass", v_zoom},
      {"speedup", v_speedup},    {"stage-shares", v_shares}};
  std::vector<std::string> run;
  if (a.target == "all") {
    for (auto& kv : cases) run.push_back(kv.first);
  } else if (cases.count(a.target)) {
    run.push_back(a.target);
  } else {
    usage("unknown validation case '" + a.target + "'");
  }
  bool all = true;
  for (auto& name : run) {
    Report r = cases[name](a);
    std::printf("%-18s %s\n", r.name.c_str(), r.pass ? "PASS" : "FAIL");
    for (auto& m : r.metrics) std::printf("    %-40s %.6g\n", m.first.c_str(), m.second);
    std::printf("    threshold: %s\n", r.threshold.c_str());
    all = all && r.pass;
  }
  return all ? 0 : 2;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    Args a = parse(argc, argv);
    if (a.cmd == "run") return cmd_run(a);
    if (a.cmd == "bench") return cmd_bench(a);
    if (a.cmd == "info") return cmd_info(a);
    return cmd_validate(a);
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "swflood: configuration error: %s\n", e.what());
    return 1;
  } catch (const NumericalError& e) {
    std::fprintf(stderr, "swflood: numerical abort: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "swflood: error: %s\n", e.what());
    return 1;
  }
}
