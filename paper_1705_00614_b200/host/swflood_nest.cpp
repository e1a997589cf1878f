// swflood_nest.cpp — C++ nesting API (include/swflood/nesting.hpp) over the
// swf_nest_* / swf_coupled_step entry points of libswflood_cuda.so.
#include "swflood/nesting.hpp"

#include <cmath>

namespace swflood {

namespace {

[[noreturn]] void throw_status(int rc, const std::string& m) {
  switch (rc) {
    case SWF_ECONFIG: throw ConfigError(m);
    case SWF_ENUMERICAL: throw NumericalError(m);
    case SWF_ERANGE: throw std::out_of_range(m);
    default: throw std::runtime_error(m);
  }
}

StepInfo from_c(const swf_step_info& c) {
  StepInfo s;
  s.tau = c.tau;
  s.active_fraction = c.active_fraction;
  s.lagrangian_blocks = c.lagrangian_blocks;
  s.flux_blocks = c.flux_blocks;
  s.total_blocks = c.total_blocks;
  s.timings = {c.timings[0], c.timings[1], c.timings[2], c.timings[3],
               c.timings[4], c.timings[5], c.timings[6], c.timings[7]};
  s.clamp_deficit_volume = c.clamp_deficit_volume;
  s.source_volume = c.source_volume;
  s.boundary_outflow_volume = c.boundary_outflow_volume;
  return s;
}

}  // namespace

NestedGrid::NestedGrid(CsphTvdStepper& global, NestWindow window, Terrain fine_terrain,
                       PhysicalParams fine_params, TimestepControl control,
                       StepperOptions options)
    : global_(&global), w_(window), terrain_(std::move(fine_terrain)) {
  if (terrain_.nx != w_.fine_nx() || terrain_.ny != w_.fine_ny())
    throw ConfigError("nest: fine terrain must be " + std::to_string(w_.fine_nx()) + "x" +
                      std::to_string(w_.fine_ny()) + " (r*window + 2*ghost)");
  fine_ = std::make_unique<CsphTvdStepper>(terrain_, std::move(fine_params), control, options);
  swf_nest_desc d{w_.i0, w_.j0, w_.ni, w_.nj, w_.r, w_.ghost, w_.two_way ? 1 : 0};
  int rc = swf_nest_create(global.native(), fine_->native(), &d, &nest_);
  if (rc) throw_status(rc, swf_last_error(global.native()));
}

NestedGrid::~NestedGrid() {
  if (nest_) swf_nest_destroy(nest_);
}

void NestedGrid::set_state(const FlowState& s) {
  if (s.nx != terrain_.nx || s.ny != terrain_.ny)
    throw ConfigError("nest: state does not match the fine grid");
  int rc = swf_upload_state(fine_->native(), s.H.data(), s.HUx.data(), s.HUy.data(), s.t);
  if (rc) throw_status(rc, swf_last_error(fine_->native()));
}

FlowState NestedGrid::state() const {
  FlowState s = FlowState::dry(terrain_);
  int rc = swf_download_state(fine_->native(), s.H.data(), s.HUx.data(), s.HUy.data(), &s.t);
  if (rc) throw_status(rc, swf_last_error(fine_->native()));
  return s;
}

std::vector<double> NestedGrid::prolong_boundary(int slot) {
  size_t n = 0;
  swf_nest_ghost_count(nest_, &n);
  std::vector<double> out(3 * n);
  int rc = swf_nest_prolong(nest_, slot);
  if (!rc) rc = swf_nest_download_ghosts(nest_, slot, out.data());
  if (rc) throw_status(rc, swf_nest_last_error(nest_));
  return out;
}

void NestedGrid::restrict_feedback() {
  int rc = swf_nest_restrict(nest_);
  if (rc) throw_status(rc, swf_nest_last_error(nest_));
}

double NestedGrid::bathymetry_deviation() const {
  const Terrain& g = global_->terrain();
  double acc = 0.0;
  int nxf = w_.fine_nx();
  for (int cj = 0; cj < w_.nj; ++cj)
    for (int ci = 0; ci < w_.ni; ++ci) {
      double s = 0.0;
      for (int b = 0; b < w_.r; ++b)
        for (int a = 0; a < w_.r; ++a)
          s += terrain_.b[(w_.ghost + ci * w_.r + a) + (size_t)(w_.ghost + cj * w_.r + b) * nxf];
      acc += std::fabs(s / (w_.r * w_.r) - g.b[g.idx(w_.i0 + ci, w_.j0 + cj)]);
    }
  return acc / (double(w_.ni) * w_.nj);
}

CoupledStepInfo coupled_step_resident(CsphTvdStepper& global, const std::vector<NestedGrid*>& nests,
                                      double dt_cap) {
  std::vector<swf_nest*> p;
  for (NestedGrid* n : nests) p.push_back(n->native());
  swf_coupled_info c{};
  int rc = swf_coupled_step(global.native(), p.data(), (int)p.size(), dt_cap, &c);
  if (rc) throw_status(rc, swf_last_error(global.native()));
  CoupledStepInfo I;
  I.tau = c.tau;
  I.substeps_total = c.substeps_total;
  I.substeps_max = c.substeps_max;
  I.fine_tau_min = c.fine_tau_min;
  I.global = from_c(c.coarse);
  I.reflux_clamp_volume = c.reflux_clamp_volume;
  return I;
}

CoupledStepInfo coupled_step(CsphTvdStepper& global, FlowState& s,
                             const std::vector<NestedGrid*>& nests, double dt_cap) {
  swf_ctx* c = global.native();
  int rc = swf_upload_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), s.t);
  if (rc) throw_status(rc, swf_last_error(c));
  CoupledStepInfo I = coupled_step_resident(global, nests, dt_cap);
  rc = swf_download_state(c, s.H.data(), s.HUx.data(), s.HUy.data(), &s.t);
  if (rc) throw_status(rc, swf_last_error(c));
  return I;
}

}  // namespace swflood
