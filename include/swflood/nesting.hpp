// swflood/nesting.hpp — two-level nested grids (SPEC.md [MODULE] nesting,
// SPEC.md:363-417).  The reference declares this module in its SPEC only (no
// header ships under proj/include), so the names follow the SPEC operations:
// NestedGrid (:366-370), prolong_boundary (:371-378), restrict_feedback
// (:379-385), coupled_step (:386-392).  Both levels run on the GPU
// (libswflood_cuda.so, csrc/swf_nest.cu); see that file for the operators.
#pragma once

#include <memory>
#include <vector>

#include "../swflood_b200.hpp"

namespace swflood {

struct NestWindow {
  int i0 = 0, j0 = 0, ni = 0, nj = 0;  // global cells [i0, i0+ni) x [j0, j0+nj)
  int r = 4;                            // refinement factor (global h / fine h)
  int ghost = 2;                        // interpolation ghost band (fine cells)
  bool two_way = true;                  // restrict_feedback after each coupled step
  int fine_nx() const { return r * ni + 2 * ghost; }
  int fine_ny() const { return r * nj + 2 * ghost; }
};

struct CoupledStepInfo {
  double tau = 0.0;          // the global step
  int substeps_total = 0;    // fine steps over all windows
  int substeps_max = 0;
  double fine_tau_min = 0.0;
  StepInfo global;
  double reflux_clamp_volume = 0.0;  // flux-correction clamp (mass ledger)
};

class NestedGrid {
 public:
  // fine_terrain: fine_nx() x fine_ny() cells at h/r (ghost band included);
  // the default options use open edges (the ghost band is rewritten each
  // substep).  Throws ConfigError for windows that do not fit.
  NestedGrid(CsphTvdStepper& global, NestWindow window, Terrain fine_terrain,
             PhysicalParams fine_params, TimestepControl control = {},
             StepperOptions options = open_edges());
  static StepperOptions open_edges() {
    StepperOptions o;
    o.boundaries = BoundaryConfig::all(EdgeKind::Open);
    return o;
  }
  ~NestedGrid();
  NestedGrid(const NestedGrid&) = delete;
  NestedGrid& operator=(const NestedGrid&) = delete;

  const NestWindow& window() const { return w_; }
  const Terrain& fine_terrain() const { return terrain_; }
  CsphTvdStepper& fine() { return *fine_; }

  // fine state (synchronized in time with the global grid before coupling)
  void set_state(const FlowState& fine_state);
  FlowState state() const;

  // SPEC operations on the device state of both levels
  std::vector<double> prolong_boundary(int slot = 0);  // [H | HUx | HUy] of the ghost band
  void restrict_feedback();
  // mean |restrict(b_fine) - b_global| over the window (SPEC.md:368 ingestion check)
  double bathymetry_deviation() const;

  swf_nest* native() const { return nest_; }

 private:
  CsphTvdStepper* global_;
  NestWindow w_;
  Terrain terrain_;
  std::unique_ptr<CsphTvdStepper> fine_;
  swf_nest* nest_ = nullptr;
};

// SPEC.md:386-392 on the DEVICE-resident states (upload them with
// NestedGrid::set_state / swf_upload_state(global.native(), ...)).
CoupledStepInfo coupled_step_resident(CsphTvdStepper& global, const std::vector<NestedGrid*>& nests,
                                      double dt_cap = 0.0);
// Drop-in form: uploads global_state, couples, downloads it (the fine states
// stay on the device; read them with NestedGrid::state()).
CoupledStepInfo coupled_step(CsphTvdStepper& global, FlowState& global_state,
                             const std::vector<NestedGrid*>& nests, double dt_cap = 0.0);

}  // namespace swflood
