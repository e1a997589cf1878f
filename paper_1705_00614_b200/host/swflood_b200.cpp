// swflood_b200.cpp — the C++ drop-in API (include/swflood_b200.hpp) over the
// C ABI of libswflood_cuda.so.  Value-type validation mirrors the reference
// (grid.cpp:13-121, sources.cpp:10-33, stepper.cpp:31-49); everything that
// touches cells is a call into the CUDA library.
#include "swflood_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numbers>

namespace swflood {

namespace {

[[noreturn]] void throw_status(int rc, const char* msg) {
  std::string m = msg ? msg : "";
  switch (rc) {
    case SWF_ECONFIG: throw ConfigError(m);
    case SWF_ENUMERICAL: throw NumericalError(m);
    case SWF_ERANGE: throw std::out_of_range(m);
    default: throw std::runtime_error(m);
  }
}

swf_control to_c(const TimestepControl& k) { return swf_control{k.courant, k.dt_max, k.dt_min}; }

swf_options to_c(const StepperOptions& o) {
  auto e = [](EdgeKind k) { return k == EdgeKind::Open ? SWF_EDGE_OPEN : SWF_EDGE_REFLECTIVE; };
  return swf_options{o.block_size, o.skip_dry_blocks ? 1 : 0, o.workers,
                     e(o.boundaries.west), e(o.boundaries.east), e(o.boundaries.south),
                     e(o.boundaries.north)};
}

bool same(const TimestepControl& a, const TimestepControl& b) {
  return a.courant == b.courant && a.dt_max == b.dt_max && a.dt_min == b.dt_min;
}

bool same(const StepperOptions& a, const StepperOptions& b) {
  return a.block_size == b.block_size && a.skip_dry_blocks == b.skip_dry_blocks &&
         a.workers == b.workers && a.boundaries.west == b.boundaries.west &&
         a.boundaries.east == b.boundaries.east && a.boundaries.south == b.boundaries.south &&
         a.boundaries.north == b.boundaries.north;
}

template <class T>
double interp_series(const std::vector<T>& s, double t, double T::*val) {
  if (s.empty()) return 0.0;
  if (s.size() == 1 || t <= s.front().t) return s.front().*val;
  if (t >= s.back().t) return s.back().*val;
  auto hi = std::upper_bound(s.begin(), s.end(), t, [](double v, const T& x) { return v < x.t; });
  const T& H = *hi;
  const T& L = *(hi - 1);
  double a = (t - L.t) / (H.t - L.t);
  return L.*val + a * (H.*val - L.*val);
}

// SourceSpecs as swf_source records (the hydrograph arrays live in `keep`)
struct CSources {
  std::vector<swf_source> v;
  std::vector<std::vector<double>> keep;
  explicit CSources(const std::vector<SourceSpec>& sources) {
    keep.reserve(2 * sources.size());
    for (const SourceSpec& s : sources) {
      keep.emplace_back();
      keep.emplace_back();
      auto& ts = keep[keep.size() - 2];
      auto& qs = keep.back();
      for (const HydrographSample& h : s.hydrograph) {
        ts.push_back(h.t);
        qs.push_back(h.q);
      }
      v.push_back(swf_source{s.kind == SourceSpec::Kind::Rain ? SWF_SOURCE_RAIN : SWF_SOURCE_DISCHARGE,
                             s.cells.i0, s.cells.j0, s.cells.i1, s.cells.j1, (int)ts.size(),
                             ts.data(), qs.data(), s.rate, s.source_velocity.x,
                             s.source_velocity.y});
    }
  }
};

swf_terrain to_c(const Terrain& t) {
  return swf_terrain{t.nx, t.ny, t.h, t.x0, t.y0, t.b.data()};
}

swf_params to_c(const PhysicalParams& p) {
  return swf_params{p.g,   p.n_manning, p.nu,        p.omega_z, p.c_a,
                    p.rho_air, p.rho_water, p.eps_dry, p.n_field.empty() ? nullptr : p.n_field.data()};
}

void check_state(const FlowState& s, const Terrain& t, const char* what) {
  if (s.nx != t.nx || s.ny != t.ny || s.H.size() != t.cells() || s.HUx.size() != t.cells() ||
      s.HUy.size() != t.cells() || t.b.size() != t.cells())
    throw ConfigError(std::string(what) + ": state does not match the terrain grid");
}

// viscous_force / surface_gradient_force at one cell: the 3x3 window around
// (i, j) clipped at the domain edges only, so every neighbour test of the
// 5-point stencil (i > 0, i + 1 < nx, ...) reads the same inside the window
Vec2 point_force(const FlowState& state, const Terrain& terrain, const PhysicalParams& params,
                 int i, int j, int which) {
  check_state(state, terrain, which == SWF_POINT_VISCOUS ? "viscous_force" : "surface_gradient_force");
  if (!terrain.contains(i, j)) throw std::out_of_range("cell index outside grid");
  const int i0 = std::max(0, i - 1), i1 = std::min(terrain.nx - 1, i + 1);
  const int j0 = std::max(0, j - 1), j1 = std::min(terrain.ny - 1, j + 1);
  const int wx = i1 - i0 + 1, wy = j1 - j0 + 1;
  std::vector<double> H, U, V, B;
  for (int jj = j0; jj <= j1; ++jj)
    for (int ii = i0; ii <= i1; ++ii) {
      const int k = terrain.idx(ii, jj);
      H.push_back(state.H[k]);
      U.push_back(state.HUx[k]);
      V.push_back(state.HUy[k]);
      B.push_back(terrain.b[k]);
    }
  // the window is a whole domain only where it touches a real edge: a stencil
  // neighbour "outside" the window is outside the grid exactly then
  swf_terrain tw{wx, wy, terrain.h, 0.0, 0.0, B.data()};
  swf_params pw = to_c(params);
  pw.n_field = nullptr;
  int ij[2] = {i - i0, j - j0};
  double out[2];
  if (int rc = swf_dev_point_forces(&tw, &pw, H.data(), U.data(), V.data(), which, 1, ij, out))
    throw_status(rc, swf_last_error(nullptr));
  return {out[0], out[1]};
}

}  // namespace

// ---- value types ------------------------------------------------------------

void Terrain::validate() const {
  if (nx < 1 || ny < 1) throw ConfigError("terrain: nx and ny must be >= 1");
  if (!(h > 0.0)) throw ConfigError("terrain: cell size must be positive");
  if (b.size() != cells()) throw ConfigError("terrain: bed array size mismatch");
  for (std::size_t k = 0; k < b.size(); ++k)
    if (!std::isfinite(b[k]))
      throw ConfigError("terrain: non-finite bed elevation at cell " + std::to_string(k));
}

FlowState FlowState::dry(const Terrain& terrain) {
  FlowState s;
  s.nx = terrain.nx;
  s.ny = terrain.ny;
  s.H.assign(terrain.cells(), 0.0);
  s.HUx.assign(terrain.cells(), 0.0);
  s.HUy.assign(terrain.cells(), 0.0);
  return s;
}

void FlowState::enforce_dry_rule(double eps_dry) {
  for (std::size_t k = 0; k < H.size(); ++k)
    if (H[k] <= eps_dry) HUx[k] = HUy[k] = 0.0;
}

void PhysicalParams::validate() const {
  if (!(g > 0.0)) throw ConfigError("params: gravity must be positive");
  if (n_manning < 0.0) throw ConfigError("params: Manning coefficient must be >= 0");
  if (std::any_of(n_field.begin(), n_field.end(), [](double n) { return n < 0.0; }))
    throw ConfigError("params: Manning field must be >= 0");
  if (nu < 0.0) throw ConfigError("params: viscosity must be >= 0");
  if (!(rho_water > 0.0)) throw ConfigError("params: water density must be positive");
  if (rho_air < 0.0) throw ConfigError("params: air density must be >= 0");
  if (!(eps_dry > 0.0)) throw ConfigError("params: dry threshold must be positive");
}

double latitude_to_omega_z(double latitude_deg) {
  return 7.2921159e-5 * std::sin(latitude_deg * std::numbers::pi / 180.0);
}

Vec2 WindForcing::at(double t) const {
  return {interp_series(series, t, &WindSample::wx), interp_series(series, t, &WindSample::wy)};
}

void WindForcing::validate() const {
  for (std::size_t k = 1; k < series.size(); ++k)
    if (!(series[k].t > series[k - 1].t))
      throw ConfigError("wind: sample times must be strictly increasing");
}

void SourceField::resize(int nx_, int ny_) {
  nx = nx_;
  ny = ny_;
  std::size_t n = std::size_t(nx_) * std::size_t(ny_);
  sigma.assign(n, 0.0);
  vx.assign(n, 0.0);
  vy.assign(n, 0.0);
  index_q.assign(n, 0);
}

void SourceField::clear_values() {
  std::fill(sigma.begin(), sigma.end(), 0.0);
  std::fill(vx.begin(), vx.end(), 0.0);
  std::fill(vy.begin(), vy.end(), 0.0);
  std::fill(index_q.begin(), index_q.end(), 0);
}

double free_surface(const FlowState& state, const Terrain& terrain, int i, int j) {
  if (!terrain.contains(i, j))
    throw std::out_of_range("free_surface: cell (" + std::to_string(i) + "," + std::to_string(j) +
                            ") outside grid");
  return state.H[state.idx(i, j)] + terrain.b[terrain.idx(i, j)];
}

Vec2 velocity(const FlowState& state, const PhysicalParams& params, int i, int j) {
  if (i < 0 || i >= state.nx || j < 0 || j >= state.ny)
    throw std::out_of_range("velocity: cell index outside grid");
  int k = state.idx(i, j);
  if (state.H[k] <= params.eps_dry) return {};
  return {state.HUx[k] / state.H[k], state.HUy[k] / state.H[k]};
}

double total_volume(const FlowState& state, const Terrain& terrain) {
  double s = 0.0;
  for (double v : state.H) s += v;
  return s * terrain.cell_area();
}

double SourceSpec::discharge_at(double t) const {
  return interp_series(hydrograph, t, &HydrographSample::q);
}

void SourceSpec::validate(const Terrain& terrain) const {
  if (cells.i0 > cells.i1 || cells.j0 > cells.j1)
    throw ConfigError("source '" + name + "': empty cell rectangle");
  if (!terrain.contains(cells.i0, cells.j0) || !terrain.contains(cells.i1, cells.j1))
    throw ConfigError("source '" + name + "': cells outside grid");
  for (std::size_t k = 1; k < hydrograph.size(); ++k)
    if (!(hydrograph[k].t > hydrograph[k - 1].t))
      throw ConfigError("source '" + name + "': hydrograph times must be strictly increasing");
  if (kind == Kind::Discharge && hydrograph.empty())
    throw ConfigError("source '" + name + "': discharge source needs a hydrograph");
}

void ForceField::resize(int nx_, int ny_) {
  nx = nx_;
  ny = ny_;
  std::size_t n = std::size_t(nx_) * std::size_t(ny_);
  for (auto* v : {&fx, &fy, &fric_x, &fric_y, &sigma_eff}) v->assign(n, 0.0);
}

void ForceField::clear() {
  for (auto* v : {&fx, &fy, &fric_x, &fric_y, &sigma_eff}) std::fill(v->begin(), v->end(), 0.0);
}

Vec2 bottom_friction(Vec2 u, double H, double g, double n_manning) {
  double in[3] = {u.x, u.y, H}, out[2];
  int rc = swf_dev_bottom_friction(1, in, g, n_manning, out);
  if (rc) throw_status(rc, swf_last_error(nullptr));
  return {out[0], out[1]};
}

Vec2 bottom_friction(Vec2 u, double H, const PhysicalParams& p) {
  return bottom_friction(u, H, p.g, p.n_manning);  // scalar n, forcing.cpp:30-32
}

FaceFlux hll_face_flux(double hL, double unL, double utL, double hR, double unR, double utR,
                       double g) {
  double in[6] = {hL, unL, utL, hR, unR, utR}, out[3];
  int rc = swf_dev_hll_face_flux(1, in, g, out);
  if (rc) throw_status(rc, swf_last_error(nullptr));
  return {out[0], out[1], out[2]};
}

Vec2 viscous_force(const FlowState& state, const PhysicalParams& params, const Terrain& terrain,
                   int i, int j) {
  return point_force(state, terrain, params, i, j, SWF_POINT_VISCOUS);
}

Vec2 coriolis_force(Vec2 u, const PhysicalParams& params) {
  double in[2] = {u.x, u.y}, out[2];
  if (int rc = swf_dev_coriolis_force(1, in, params.omega_z, out))
    throw_status(rc, swf_last_error(nullptr));
  return {out[0], out[1]};
}

Vec2 wind_force(Vec2 u, double H, const WindForcing& wind, double t, const PhysicalParams& params) {
  const Vec2 w = wind.at(t);  // host: the series lookup (grid.cpp:64-75)
  double in[3] = {u.x, u.y, H}, out[2];
  swf_params p = to_c(params);
  if (int rc = swf_dev_wind_force(1, in, w.x, w.y, &p, out)) throw_status(rc, swf_last_error(nullptr));
  return {out[0], out[1]};
}

Vec2 surface_gradient_force(const FlowState& state, const Terrain& terrain,
                            const PhysicalParams& params, int i, int j) {
  return point_force(state, terrain, params, i, j, SWF_POINT_SURFACE_GRADIENT);
}

ForceField assemble_forces(const FlowState& state, const Terrain& terrain,
                           const PhysicalParams& params, const WindForcing& wind,
                           const SourceField& src, double t) {
  check_state(state, terrain, "assemble_forces");
  if (!params.n_field.empty() && params.n_field.size() != terrain.cells())
    throw ConfigError("assemble_forces: Manning field size mismatch");
  const bool present = !src.empty();
  if (present && (src.sigma.size() != terrain.cells() || src.vx.size() != terrain.cells() ||
                  src.vy.size() != terrain.cells()))
    throw ConfigError("assemble_forces: source field size mismatch");
  ForceField out;
  out.resize(terrain.nx, terrain.ny);
  const Vec2 w = wind.at(t);
  swf_terrain T = to_c(terrain);
  swf_params P = to_c(params);
  if (int rc = swf_dev_assemble_forces(&T, &P, state.H.data(), state.HUx.data(), state.HUy.data(),
                                       wind.any() ? 1 : 0, w.x, w.y,
                                       present ? src.sigma.data() : nullptr,
                                       present ? src.vx.data() : nullptr,
                                       present ? src.vy.data() : nullptr, out.fx.data(),
                                       out.fy.data(), out.fric_x.data(), out.fric_y.data(),
                                       out.sigma_eff.data()))
    throw_status(rc, swf_last_error(nullptr));
  return out;
}

SourceField source_terms(const std::vector<SourceSpec>& sources, double t, const Terrain& terrain) {
  for (const SourceSpec& s : sources) s.validate(terrain);  // sources.cpp:48
  SourceField f;
  f.resize(terrain.nx, terrain.ny);
  CSources cs(sources);
  swf_terrain T = to_c(terrain);
  if (int rc = swf_dev_source_terms(&T, cs.v.data(), (int)cs.v.size(), t, 0, f.sigma.data(),
                                    f.vx.data(), f.vy.data(), f.index_q.data()))
    throw_status(rc, swf_last_error(nullptr));
  return f;
}

void resample_sigma(const std::vector<SourceSpec>& sources, double t, const Terrain& terrain,
                    SourceField& field) {
  if (field.sigma.size() != terrain.cells()) field.sigma.assign(terrain.cells(), 0.0);
  CSources cs(sources);
  swf_terrain T = to_c(terrain);
  if (int rc = swf_dev_source_terms(&T, cs.v.data(), (int)cs.v.size(), t, 1, field.sigma.data(),
                                    nullptr, nullptr, nullptr))
    throw_status(rc, swf_last_error(nullptr));
}

BlockMask compute_block_mask(const FlowState& state, const SourceField& sources, double eps_dry,
                             int block_size) {
  if (block_size < 1) throw ConfigError("block mask: block size must be >= 1");
  if (state.H.size() != state.cells()) throw ConfigError("block mask: state size mismatch");
  const bool has_src = !sources.empty();
  if (has_src && sources.index_q.size() != state.cells())
    throw ConfigError("block mask: source field size mismatch");
  BlockMask m;
  m.block_size = block_size;
  m.nx = state.nx;
  m.ny = state.ny;
  m.nbx = (state.nx + block_size - 1) / block_size;
  m.nby = (state.ny + block_size - 1) / block_size;
  m.interior_wet.assign(m.total_blocks(), 0);
  m.halo_wet.assign(m.total_blocks(), 0);
  if (m.total_blocks() == 0) return m;
  if (int rc = swf_dev_block_mask(state.nx, state.ny, state.H.data(),
                                  has_src ? sources.index_q.data() : nullptr, eps_dry, block_size,
                                  m.interior_wet.data(), m.halo_wet.data()))
    throw_status(rc, swf_last_error(nullptr));
  return m;
}

// block.cpp:63-79: dispatch over the mask (host control flow; the bodies are
// the caller's)
void for_each_active_block(const BlockMask& mask, StageKind kind,
                           const std::function<void(int)>& body,
                           const std::function<void(int)>& skipped) {
  for (int ib = 0; ib < mask.total_blocks(); ++ib) {
    if (mask.active(ib, kind))
      body(ib);
    else if (skipped)
      skipped(ib);
  }
}

std::vector<int> active_blocks(const BlockMask& mask, StageKind kind) {
  std::vector<int> out;
  for (int ib = 0; ib < mask.total_blocks(); ++ib)
    if (mask.active(ib, kind)) out.push_back(ib);
  return out;
}

void BlockMask::block_rect(int ib, int& i0, int& j0, int& i1, int& j1) const {
  i0 = (ib % nbx) * block_size;
  j0 = (ib / nbx) * block_size;
  i1 = std::min(i0 + block_size - 1, nx - 1);
  j1 = std::min(j0 + block_size - 1, ny - 1);
}

double active_fraction(const BlockMask& m) {
  if (m.total_blocks() == 0) return 0.0;
  int n = 0;
  for (int ib = 0; ib < m.total_blocks(); ++ib) n += m.flux_active(ib);
  return static_cast<double>(n) / m.total_blocks();
}

void TimestepControl::validate() const {
  if (!(courant > 0.0 && courant < 1.0)) throw ConfigError("timestep: Courant number must be in (0,1)");
  if (!(dt_max > 0.0)) throw ConfigError("timestep: dt_max must be positive");
  if (!(dt_min > 0.0 && dt_min < dt_max)) throw ConfigError("timestep: need 0 < dt_min < dt_max");
}

StageTimings& StageTimings::operator+=(const StageTimings& o) {
  mask += o.mask;
  forces += o.forces;
  dt += o.dt;
  predictor += o.predictor;
  mid_forces += o.mid_forces;
  corrector += o.corrector;
  flux += o.flux;
  finalize += o.finalize;
  return *this;
}

// ---- the stepper --------------------------------------------------------------

CsphTvdStepper::CsphTvdStepper(const Terrain& terrain, PhysicalParams params,
                               TimestepControl control, StepperOptions options)
    : terrain_(&terrain), params_(std::move(params)), ctl_(control), opt_(options) {
  terrain.validate();
  params_.validate();
  ctl_.validate();
  if (opt_.block_size < 1) throw ConfigError("stepper: block size must be >= 1");
  if (opt_.workers < 1) opt_.workers = 1;
  if (!params_.n_field.empty() && params_.n_field.size() != terrain.cells())
    throw ConfigError("stepper: Manning field size mismatch");
  if (opt_.devices < 1) throw ConfigError("stepper: devices must be >= 1");
  create();
}

// the device context(s) for the current configuration
void CsphTvdStepper::create() {
  const Terrain& terrain = *terrain_;
  swf_terrain t = to_c(terrain);
  swf_params p = to_c(params_);
  swf_control k = to_c(ctl_);
  swf_options o = to_c(opt_);
  if (opt_.devices == 1) {
    int rc = swf_create(&t, &p, &k, &o, &ctx_);
    if (rc) throw_status(rc, swf_last_error(nullptr));
  } else {
    // row strips on block boundaries, one per device, windows of the global arrays
    const int D = opt_.devices, bs = opt_.block_size, nby = (terrain.ny + bs - 1) / bs;
    if (D > nby) throw ConfigError("stepper: more devices than block rows");
    int ndev = 0;
    int rc = swf_device_count(&ndev);
    if (rc || ndev < 1) throw_status(rc ? rc : SWF_ECUDA, swf_last_error(nullptr));
    // block-row cuts, then every strip at least SWF_HALO rows (a neighbour's
    // ghost rows come from one strip's owned rows; multigpu.min_rows_cuts)
    std::vector<int> cut(D + 1);
    for (int d = 0; d <= D; ++d) cut[d] = (int)((long long)d * nby / D);
    auto rows = [&](int d) {
      return std::min(terrain.ny, cut[d + 1] * bs) - std::min(terrain.ny, cut[d] * bs);
    };
    if (D > 1) {
      for (int d = D - 1; d > 0; --d)
        while (rows(d) < SWF_HALO && cut[d] - 1 > cut[d - 1]) --cut[d];
      for (int d = 0; d + 1 < D; ++d)
        while (rows(d) < SWF_HALO && cut[d + 1] + 1 < cut[d + 2]) ++cut[d + 1];
      for (int d = 0; d < D; ++d)
        if (rows(d) < SWF_HALO) throw ConfigError("stepper: too many devices for the grid rows");
    }
    for (int d = 0; d < D; ++d) {
      int j0 = std::min(terrain.ny, cut[d] * bs);
      int j1 = std::min(terrain.ny, cut[d + 1] * bs);
      int w0 = std::max(0, j0 - SWF_HALO);
      swf_terrain tw = t;
      tw.b = terrain.b.data() + (size_t)w0 * terrain.nx;
      swf_params pw = p;
      if (pw.n_field) pw.n_field = params_.n_field.data() + (size_t)w0 * terrain.nx;
      swf_ctx* c = nullptr;
      rc = swf_create_strip(&tw, &pw, &k, &o, j0, j1, d % ndev, &c);
      if (rc) {
        std::string m = swf_last_error(nullptr);
        for (swf_ctx* s : strips_) swf_destroy(s);
        strips_.clear();
        throw_status(rc, m.c_str());
      }
      strips_.push_back(c);
    }
    rc = swf_group_create(strips_.data(), D, &group_);
    if (rc) {
      std::string m = swf_last_error(nullptr);
      for (swf_ctx* s : strips_) swf_destroy(s);
      strips_.clear();
      throw_status(rc, m.c_str());
    }
    ctx_ = strips_[0];
  }
  pushed_ctl_ = ctl_;
  pushed_opt_ = opt_;
}

void CsphTvdStepper::release() noexcept {
  if (group_) {
    swf_group_destroy(group_);
    for (swf_ctx* s : strips_) swf_destroy(s);
  } else if (ctx_) {
    swf_destroy(ctx_);
  }
  group_ = nullptr;
  strips_.clear();
  ctx_ = nullptr;
}

CsphTvdStepper::~CsphTvdStepper() { release(); }

CsphTvdStepper::CsphTvdStepper(const CsphTvdStepper& o)
    : terrain_(o.terrain_), params_(o.params_), ctl_(o.ctl_), opt_(o.opt_) {
  create();
  try {
    if (o.wind_.any()) set_wind(o.wind_);
    if (!o.sources_.empty()) set_sources(o.sources_);
  } catch (...) {
    release();
    throw;
  }
}

CsphTvdStepper& CsphTvdStepper::operator=(const CsphTvdStepper& o) {
  if (this != &o) {
    CsphTvdStepper tmp(o);
    swap(tmp);
  }
  return *this;
}

CsphTvdStepper::CsphTvdStepper(CsphTvdStepper&& o) noexcept
    : terrain_(o.terrain_), params_(o.params_), ctl_(o.ctl_), opt_(o.opt_) {
  swap(o);
}

CsphTvdStepper& CsphTvdStepper::operator=(CsphTvdStepper&& o) noexcept {
  if (this != &o) {
    release();
    swap(o);
  }
  return *this;
}

void CsphTvdStepper::swap(CsphTvdStepper& o) noexcept {
  using std::swap;
  swap(terrain_, o.terrain_);
  swap(params_, o.params_);
  swap(ctl_, o.ctl_);
  swap(opt_, o.opt_);
  swap(wind_, o.wind_);
  swap(sources_, o.sources_);
  swap(ctx_, o.ctx_);
  swap(strips_, o.strips_);
  swap(group_, o.group_);
  swap(group_vol_, o.group_vol_);
  swap(pushed_ctl_, o.pushed_ctl_);
  swap(pushed_opt_, o.pushed_opt_);
  swap(mask_, o.mask_);
  swap(src_, o.src_);
  swap(f_n_, o.f_n_);
  swap(f_mid_, o.f_mid_);
  for (int q = 0; q < 9; ++q) swap(buf_[q], o.buf_[q]);
}

std::vector<swf_ctx*> CsphTvdStepper::contexts() const {
  return group_ ? strips_ : std::vector<swf_ctx*>{ctx_};
}

void CsphTvdStepper::single(const char* what) const {
  if (group_)
    throw ConfigError(std::string("stepper: ") + what + " needs StepperOptions::devices == 1");
}

void CsphTvdStepper::check(int rc) const {
  if (rc) throw_status(rc, swf_last_error(ctx_));
}

void CsphTvdStepper::sync_config() const {
  if (!same(ctl_, pushed_ctl_)) {
    swf_control k = to_c(ctl_);
    for (swf_ctx* c : contexts())
      if (int rc = swf_set_control(c, &k)) throw_status(rc, swf_last_error(c));
    pushed_ctl_ = ctl_;
  }
  if (!same(opt_, pushed_opt_)) {
    swf_options o = to_c(opt_);
    for (swf_ctx* c : contexts())
      if (int rc = swf_set_options(c, &o)) throw_status(rc, swf_last_error(c));
    pushed_opt_ = opt_;
  }
}

void CsphTvdStepper::set_wind(WindForcing wind) {
  wind.validate();
  std::vector<double> t, x, y;
  for (const WindSample& s : wind.series) {
    t.push_back(s.t);
    x.push_back(s.wx);
    y.push_back(s.wy);
  }
  for (swf_ctx* c : contexts())
    if (int rc = swf_set_wind(c, (int)t.size(), t.data(), x.data(), y.data()))
      throw_status(rc, swf_last_error(c));
  wind_ = std::move(wind);
}

void CsphTvdStepper::set_host_mirror(bool on) {
  for (swf_ctx* c : contexts()) check(swf_set_host_mirror(c, on ? 1 : 0));
}

void CsphTvdStepper::host_changed() {
  for (swf_ctx* c : contexts()) check(swf_host_changed(c));
}

void CsphTvdStepper::set_sources(std::vector<SourceSpec> sources) {
  for (const SourceSpec& s : sources) s.validate(*terrain_);
  CSources cs(sources);
  for (swf_ctx* c : contexts())
    if (int rc = swf_set_sources(c, (int)cs.v.size(), cs.v.data())) throw_status(rc, swf_last_error(c));
  sources_ = std::move(sources);
}

StepInfo CsphTvdStepper::step(FlowState& state, double dt_cap) {
  if (state.nx != terrain_->nx || state.ny != terrain_->ny)
    throw ConfigError("stepper: state does not match the terrain grid");
  sync_config();
  if (group_) return step_group(state, dt_cap);
  swf_step_info ci{};
  check(swf_step_host(ctx_, state.H.data(), state.HUx.data(), state.HUy.data(), &state.t, dt_cap,
                      &ci));
  StepInfo s;
  s.tau = ci.tau;
  s.active_fraction = ci.active_fraction;
  s.lagrangian_blocks = ci.lagrangian_blocks;
  s.flux_blocks = ci.flux_blocks;
  s.total_blocks = ci.total_blocks;
  double* tm[8] = {&s.timings.mask,       &s.timings.forces,    &s.timings.dt,
                   &s.timings.predictor,  &s.timings.mid_forces, &s.timings.corrector,
                   &s.timings.flux,       &s.timings.finalize};
  for (int q = 0; q < 8; ++q) *tm[q] = ci.timings[q];
  s.clamp_deficit_volume = ci.clamp_deficit_volume;
  s.source_volume = ci.source_volume;
  s.boundary_outflow_volume = ci.boundary_outflow_volume;
  return s;
}

// devices > 1: every strip uploads its window (owned + ghost rows) straight
// from the caller's arrays, the group steps once, the owned rows come back;
// on an error the caller's state is untouched
StepInfo CsphTvdStepper::step_group(FlowState& state, double dt_cap) {
  const size_t nx = (size_t)terrain_->nx;
  for (swf_ctx* c : strips_) {
    int j0, j1, glo, ghi;
    swf_strip_rows(c, &j0, &j1, &glo, &ghi);
    size_t off = (size_t)(j0 - glo) * nx;
    if (int rc = swf_upload_state(c, state.H.data() + off, state.HUx.data() + off,
                                  state.HUy.data() + off, state.t))
      throw_status(rc, swf_last_error(c));
  }
  int done = 0;
  swf_step_info ci{};
  if (int rc = swf_group_run(group_, 1, dt_cap, &done, &ci))
    throw_status(rc, swf_group_last_error(group_));
  std::vector<double> h, x, y;
  double t = state.t;
  for (swf_ctx* c : strips_) {
    int j0, j1, glo, ghi;
    swf_strip_rows(c, &j0, &j1, &glo, &ghi);
    size_t rows = (size_t)(glo + (j1 - j0) + ghi), own = (size_t)(j1 - j0) * nx;
    h.resize(rows * nx);
    x.resize(rows * nx);
    y.resize(rows * nx);
    if (int rc = swf_download_state(c, h.data(), x.data(), y.data(), &t))
      throw_status(rc, swf_last_error(c));
    size_t src = (size_t)glo * nx, dst = (size_t)j0 * nx;
    std::copy(h.begin() + src, h.begin() + src + own, state.H.begin() + dst);
    std::copy(x.begin() + src, x.begin() + src + own, state.HUx.begin() + dst);
    std::copy(y.begin() + src, y.begin() + src + own, state.HUy.begin() + dst);
  }
  state.t = t;
  StepInfo s;
  s.tau = ci.tau;
  s.active_fraction = ci.active_fraction;
  s.lagrangian_blocks = ci.lagrangian_blocks;
  s.flux_blocks = ci.flux_blocks;
  s.total_blocks = ci.total_blocks;
  s.clamp_deficit_volume = group_vol_[0] = ci.clamp_deficit_volume;
  s.source_volume = group_vol_[1] = ci.source_volume;
  s.boundary_outflow_volume = group_vol_[2] = ci.boundary_outflow_volume;
  return s;
}

void CsphTvdStepper::begin_step(const FlowState& state) {
  single("the stage API");
  if (state.nx != terrain_->nx || state.ny != terrain_->ny)
    throw ConfigError("stepper: state does not match the terrain grid");
  sync_config();
  check(swf_upload_state(ctx_, state.H.data(), state.HUx.data(), state.HUy.data(), state.t));
  check(swf_stage(ctx_, SWF_STAGE_BEGIN, 0.0, nullptr));
}

void CsphTvdStepper::compute_forces(const FlowState&) { single("the stage API"); check(swf_stage(ctx_, SWF_STAGE_FORCES, 0.0, nullptr)); }

double CsphTvdStepper::compute_dt(const FlowState&, double dt_cap) const {
  single("the stage API");
  double tau = 0.0;
  check(swf_stage(ctx_, SWF_STAGE_DT, dt_cap, &tau));
  return tau;
}

void CsphTvdStepper::predictor(const FlowState&, double tau) { single("the stage API"); check(swf_stage(ctx_, SWF_STAGE_PREDICTOR, tau, nullptr)); }
void CsphTvdStepper::mid_forces(const FlowState&, double tau) { single("the stage API"); check(swf_stage(ctx_, SWF_STAGE_MID_FORCES, tau, nullptr)); }
void CsphTvdStepper::corrector(const FlowState&, double tau) { single("the stage API"); check(swf_stage(ctx_, SWF_STAGE_CORRECTOR, tau, nullptr)); }
void CsphTvdStepper::flux(const FlowState&, double tau) { single("the stage API"); check(swf_stage(ctx_, SWF_STAGE_FLUX, tau, nullptr)); }

void CsphTvdStepper::final_update(FlowState& state, double tau) {
  single("the stage API");
  check(swf_stage(ctx_, SWF_STAGE_FINAL, tau, nullptr));
  check(swf_download_state(ctx_, state.H.data(), state.HUx.data(), state.HUy.data(), &state.t));
}

std::span<const double> CsphTvdStepper::scratch(int which, std::vector<double>& buf) const {
  single("the scratch accessors");
  buf.resize(terrain_->cells());
  check(swf_download_scratch(ctx_, which, buf.data()));
  return buf;
}

const BlockMask& CsphTvdStepper::mask() const {
  single("mask()");
  int nbx = 0, nby = 0;
  check(swf_download_mask(ctx_, nullptr, nullptr, &nbx, &nby));
  mask_.block_size = opt_.block_size;
  mask_.nx = terrain_->nx;
  mask_.ny = terrain_->ny;
  mask_.nbx = nbx;
  mask_.nby = nby;
  mask_.interior_wet.resize(std::size_t(nbx) * nby);
  mask_.halo_wet.resize(std::size_t(nbx) * nby);
  check(swf_download_mask(ctx_, mask_.interior_wet.data(), mask_.halo_wet.data(), &nbx, &nby));
  return mask_;
}

const SourceField& CsphTvdStepper::step_sources() const {
  single("the scratch accessors");
  src_.resize(terrain_->nx, terrain_->ny);
  check(swf_download_scratch(ctx_, SWF_SCR_SIGMA, src_.sigma.data()));
  check(swf_download_scratch(ctx_, SWF_SCR_SRC_VX, src_.vx.data()));
  check(swf_download_scratch(ctx_, SWF_SCR_SRC_VY, src_.vy.data()));
  for (std::size_t k = 0; k < src_.sigma.size(); ++k) src_.index_q[k] = src_.sigma[k] != 0.0;
  return src_;
}

const ForceField& CsphTvdStepper::forces_n() const {
  single("the scratch accessors");
  f_n_.resize(terrain_->nx, terrain_->ny);
  check(swf_download_scratch(ctx_, SWF_SCR_FN_FX, f_n_.fx.data()));
  check(swf_download_scratch(ctx_, SWF_SCR_FN_FY, f_n_.fy.data()));
  check(swf_download_scratch(ctx_, SWF_SCR_FN_FRIC_X, f_n_.fric_x.data()));
  check(swf_download_scratch(ctx_, SWF_SCR_FN_FRIC_Y, f_n_.fric_y.data()));
  check(swf_download_scratch(ctx_, SWF_SCR_FN_SIGMA, f_n_.sigma_eff.data()));
  return f_n_;
}

const ForceField& CsphTvdStepper::forces_mid() const {
  single("the scratch accessors");
  f_mid_.resize(terrain_->nx, terrain_->ny);
  check(swf_download_scratch(ctx_, SWF_SCR_FM_FX, f_mid_.fx.data()));
  check(swf_download_scratch(ctx_, SWF_SCR_FM_FY, f_mid_.fy.data()));
  check(swf_download_scratch(ctx_, SWF_SCR_FM_FRIC_X, f_mid_.fric_x.data()));
  check(swf_download_scratch(ctx_, SWF_SCR_FM_FRIC_Y, f_mid_.fric_y.data()));
  check(swf_download_scratch(ctx_, SWF_SCR_FM_SIGMA, f_mid_.sigma_eff.data()));
  return f_mid_;
}

std::span<const double> CsphTvdStepper::half_depth() const { return scratch(SWF_SCR_HALF_H, buf_[0]); }
std::span<const double> CsphTvdStepper::lagrangian_depth() const { return scratch(SWF_SCR_HT, buf_[1]); }
std::span<const double> CsphTvdStepper::lagrangian_momentum_x() const { return scratch(SWF_SCR_HVTX, buf_[2]); }
std::span<const double> CsphTvdStepper::lagrangian_momentum_y() const { return scratch(SWF_SCR_HVTY, buf_[3]); }
std::span<const double> CsphTvdStepper::displacement_x() const { return scratch(SWF_SCR_DRX, buf_[4]); }
std::span<const double> CsphTvdStepper::displacement_y() const { return scratch(SWF_SCR_DRY, buf_[5]); }
std::span<const double> CsphTvdStepper::flux_mass() const { return scratch(SWF_SCR_FH, buf_[6]); }
std::span<const double> CsphTvdStepper::flux_momentum_x() const { return scratch(SWF_SCR_FVX, buf_[7]); }
std::span<const double> CsphTvdStepper::flux_momentum_y() const { return scratch(SWF_SCR_FVY, buf_[8]); }

double CsphTvdStepper::last_clamp_deficit() const {
  if (group_) return group_vol_[0];
  double v = 0.0;
  check(swf_last_volumes(ctx_, &v, nullptr, nullptr));
  return v;
}
double CsphTvdStepper::last_source_volume() const {
  if (group_) return group_vol_[1];
  double v = 0.0;
  check(swf_last_volumes(ctx_, nullptr, &v, nullptr));
  return v;
}
double CsphTvdStepper::last_boundary_outflow() const {
  if (group_) return group_vol_[2];
  double v = 0.0;
  check(swf_last_volumes(ctx_, nullptr, nullptr, &v));
  return v;
}

}  // namespace swflood
