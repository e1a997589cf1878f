// swflood_b200.hpp — C++ drop-in for the reference's solver API, backed by
// the B200 kernels of libswflood_cuda.so through the C ABI (swf.h).
//
// A program written against the reference headers
//   #include "swflood/stepper.hpp"      (proj/include/swflood/*.hpp)
// builds unchanged against include/swflood/*.hpp of this repository (thin
// forwarders to this file) and links libswflood_b200.so instead of the
// reference library.  Names, field order, defaults and exceptions follow
// the reference: grid.hpp:10-121, sources.hpp:11-46, forcing.hpp:16-57,
// riemann.hpp:7-19, block.hpp:14-52, stepper.hpp:13-169, errors.hpp:10-21.
// Value types and their validate() rules are host code (configuration); all
// per-cell arithmetic runs on the GPU.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "swf.h"

namespace swflood {

// ---- errors (errors.hpp) ---------------------------------------------------
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};

// ---- grid and state (grid.hpp) --------------------------------------------
struct Vec2 {
  double x = 0.0, y = 0.0;
};

struct Terrain {
  int nx = 0, ny = 0;
  double h = 0.0, x0 = 0.0, y0 = 0.0;
  std::vector<double> b;
  std::size_t cells() const { return std::size_t(nx) * std::size_t(ny); }
  int idx(int i, int j) const { return j * nx + i; }
  bool contains(int i, int j) const { return 0 <= i && i < nx && 0 <= j && j < ny; }
  double cell_area() const { return h * h; }
  double xc(int i) const { return x0 + (i + 0.5) * h; }
  double yc(int j) const { return y0 + (j + 0.5) * h; }
  void validate() const;
};

struct FlowState {
  int nx = 0, ny = 0;
  double t = 0.0;
  std::vector<double> H, HUx, HUy;
  static FlowState dry(const Terrain& terrain);
  std::size_t cells() const { return std::size_t(nx) * std::size_t(ny); }
  int idx(int i, int j) const { return j * nx + i; }
  void enforce_dry_rule(double eps_dry);
};

struct PhysicalParams {
  double g = 9.81, n_manning = 0.02;
  std::vector<double> n_field;
  double nu = 0.0, omega_z = 0.0, c_a = 1.0e-3, rho_air = 1.2, rho_water = 1000.0;
  double eps_dry = 1.0e-6;
  double manning(int cell) const { return n_field.empty() ? n_manning : n_field[cell]; }
  void validate() const;
};

double latitude_to_omega_z(double latitude_deg);

struct WindSample {
  double t = 0.0, wx = 0.0, wy = 0.0;
};
struct WindForcing {
  std::vector<WindSample> series;
  static WindForcing constant(double wx, double wy) { return WindForcing{{{0.0, wx, wy}}}; }
  Vec2 at(double t) const;
  bool any() const { return !series.empty(); }
  void validate() const;
};

struct SourceField {
  int nx = 0, ny = 0;
  std::vector<double> sigma, vx, vy;
  std::vector<std::uint8_t> index_q;
  void resize(int nx_, int ny_);
  void clear_values();
  bool empty() const { return sigma.empty(); }
};

double free_surface(const FlowState& state, const Terrain& terrain, int i, int j);
Vec2 velocity(const FlowState& state, const PhysicalParams& params, int i, int j);
double total_volume(const FlowState& state, const Terrain& terrain);

// ---- sources (sources.hpp) ------------------------------------------------
struct CellRect {
  int i0 = 0, j0 = 0, i1 = 0, j1 = 0;
  int count() const { return (i1 - i0 + 1) * (j1 - j0 + 1); }
};
struct HydrographSample {
  double t = 0.0, q = 0.0;
};
struct SourceSpec {
  enum class Kind { Discharge, Rain };
  Kind kind = Kind::Discharge;
  std::string name;
  CellRect cells;
  std::vector<HydrographSample> hydrograph;
  double rate = 0.0;
  Vec2 source_velocity;
  double discharge_at(double t) const;
  void validate(const Terrain& terrain) const;
};
// sources.hpp:40-46 (the per-cell fill on the GPU)
SourceField source_terms(const std::vector<SourceSpec>& sources, double t, const Terrain& terrain);
void resample_sigma(const std::vector<SourceSpec>& sources, double t, const Terrain& terrain,
                    SourceField& field);

// ---- forcing / riemann free functions (evaluated on the GPU) --------------
struct ForceField {
  int nx = 0, ny = 0;
  std::vector<double> fx, fy, fric_x, fric_y, sigma_eff;
  void resize(int nx_, int ny_);
  void clear();
};
Vec2 bottom_friction(Vec2 u, double H, double g, double n_manning);
Vec2 bottom_friction(Vec2 u, double H, const PhysicalParams& params);
// forcing.hpp:34-57 (per-cell arithmetic on the GPU, swf_dev_* in swf.h)
Vec2 viscous_force(const FlowState& state, const PhysicalParams& params, const Terrain& terrain,
                   int i, int j);
Vec2 coriolis_force(Vec2 u, const PhysicalParams& params);
Vec2 wind_force(Vec2 u, double H, const WindForcing& wind, double t, const PhysicalParams& params);
Vec2 surface_gradient_force(const FlowState& state, const Terrain& terrain,
                            const PhysicalParams& params, int i, int j);
ForceField assemble_forces(const FlowState& state, const Terrain& terrain,
                           const PhysicalParams& params, const WindForcing& wind,
                           const SourceField& src, double t);

struct FaceFlux {
  double fm = 0.0, fn = 0.0, ft = 0.0;
};
FaceFlux hll_face_flux(double hL, double unL, double utL, double hR, double unR, double utR,
                       double g);

// ---- block mask (block.hpp) -----------------------------------------------
enum class StageKind { Lagrangian, Flux, Final };
struct BlockMask {
  int block_size = 16, nbx = 0, nby = 0, nx = 0, ny = 0;
  std::vector<int> interior_wet, halo_wet;
  int total_blocks() const { return nbx * nby; }
  bool lagrangian_active(int ib) const { return interior_wet[ib] > 0; }
  bool flux_active(int ib) const { return interior_wet[ib] > 0 || halo_wet[ib] > 0; }
  bool active(int ib, StageKind k) const {
    return k == StageKind::Lagrangian ? lagrangian_active(ib) : flux_active(ib);
  }
  void block_rect(int ib, int& i0, int& j0, int& i1, int& j1) const;
};
// block.hpp:38-52 (the counts on the GPU; the dispatch is host control flow)
BlockMask compute_block_mask(const FlowState& state, const SourceField& sources, double eps_dry,
                             int block_size);
void for_each_active_block(const BlockMask& mask, StageKind kind,
                           const std::function<void(int)>& body,
                           const std::function<void(int)>& skipped = {});
std::vector<int> active_blocks(const BlockMask& mask, StageKind kind);
double active_fraction(const BlockMask& mask);

// ---- stepper (stepper.hpp) ------------------------------------------------
struct TimestepControl {
  double courant = 0.5, dt_max = 10.0, dt_min = 1e-9;
  void validate() const;
};
enum class EdgeKind { Reflective, Open };
struct BoundaryConfig {
  EdgeKind west = EdgeKind::Reflective, east = EdgeKind::Reflective;
  EdgeKind south = EdgeKind::Reflective, north = EdgeKind::Reflective;
  static BoundaryConfig all(EdgeKind k) { return {k, k, k, k}; }
};
struct StageTimings {
  double mask = 0, forces = 0, dt = 0, predictor = 0, mid_forces = 0, corrector = 0, flux = 0,
         finalize = 0;
  double total() const {
    return mask + forces + dt + predictor + mid_forces + corrector + flux + finalize;
  }
  StageTimings& operator+=(const StageTimings& o);
};
struct StepInfo {
  double tau = 0.0, active_fraction = 0.0;
  int lagrangian_blocks = 0, flux_blocks = 0, total_blocks = 0;
  StageTimings timings;
  double clamp_deficit_volume = 0.0, source_volume = 0.0, boundary_outflow_volume = 0.0;
};
struct StepperOptions {
  int block_size = 16;
  bool skip_dry_blocks = true;
  int workers = 1;  // accepted, unused on the GPU
  BoundaryConfig boundaries;
  // GPUs this stepper drives from the calling process (row strips, one per
  // device, linked by peer access).  > 1 supports step(),
  // set_wind/set_sources and control()/options(); the stage API and the
  // scratch accessors need 1.  Fixed at construction.
  int devices = 1;
};

class CsphTvdStepper {
 public:
  CsphTvdStepper(const Terrain& terrain, PhysicalParams params, TimestepControl control,
                 StepperOptions options = {});
  ~CsphTvdStepper();
  // Copyable like the reference class (stepper.hpp:76, implicitly copyable):
  // a copy owns a new device context built from the same terrain (by
  // pointer, as in the reference), parameters, control, options, wind and
  // sources, so step() on a copy gives the same results as on the original.
  // The scratch accessors of a copy (mask(), forces_n(), the spans, last_*)
  // describe the copy's own last step: empty until it has stepped.
  CsphTvdStepper(const CsphTvdStepper& other);
  CsphTvdStepper& operator=(const CsphTvdStepper& other);
  CsphTvdStepper(CsphTvdStepper&& other) noexcept;
  CsphTvdStepper& operator=(CsphTvdStepper&& other) noexcept;

  void set_wind(WindForcing wind);
  void set_sources(std::vector<SourceSpec> sources);

  StepInfo step(FlowState& state, double dt_cap = 0.0);

  // stage interface; begin_step uploads `state`, final_update writes it back
  void begin_step(const FlowState& state);
  void compute_forces(const FlowState& state);
  double compute_dt(const FlowState& state, double dt_cap = 0.0) const;
  void predictor(const FlowState& state, double tau);
  void mid_forces(const FlowState& state, double tau);
  void corrector(const FlowState& state, double tau);
  void flux(const FlowState& state, double tau);
  void final_update(FlowState& state, double tau);

  const Terrain& terrain() const { return *terrain_; }
  const PhysicalParams& params() const { return params_; }
  // mutable in the reference; changes are pushed to the device before the
  // next step (see sync_config)
  TimestepControl& control() { return ctl_; }
  StepperOptions& options() { return opt_; }
  const BlockMask& mask() const;
  const SourceField& step_sources() const;
  const ForceField& forces_n() const;
  const ForceField& forces_mid() const;
  std::span<const double> half_depth() const;
  std::span<const double> lagrangian_depth() const;
  std::span<const double> lagrangian_momentum_x() const;
  std::span<const double> lagrangian_momentum_y() const;
  std::span<const double> displacement_x() const;
  std::span<const double> displacement_y() const;
  std::span<const double> flux_mass() const;
  std::span<const double> flux_momentum_x() const;
  std::span<const double> flux_momentum_y() const;
  double last_clamp_deficit() const;
  double last_source_volume() const;
  double last_boundary_outflow() const;

  struct HalfView;  // stepper.hpp:121 (the half-step view lives on the device here)

  // Opt-in host mirror (swf_set_host_mirror, SURVEY.md 8b "Ownership"):
  // step() on the same FlowState, with its arrays in pinned memory, skips the
  // host->device copies as long as the caller changes the state only through
  // step(); host_changed() declares an edit.  Off by default.
  void set_host_mirror(bool on);
  void host_changed();

  swf_ctx* native() const { return ctx_; }  // the C-ABI context (resident API; strip 0 if devices > 1)

 private:
  void check(int rc) const;
  void sync_config() const;
  void single(const char* what) const;
  std::vector<swf_ctx*> contexts() const;
  StepInfo step_group(FlowState& state, double dt_cap);
  std::span<const double> scratch(int which, std::vector<double>& buf) const;

  void create();
  void release() noexcept;
  void swap(CsphTvdStepper& other) noexcept;

  const Terrain* terrain_;
  PhysicalParams params_;
  TimestepControl ctl_;
  StepperOptions opt_;
  WindForcing wind_;                  // as last set (replayed into a copy)
  std::vector<SourceSpec> sources_;
  swf_ctx* ctx_ = nullptr;
  std::vector<swf_ctx*> strips_;  // devices > 1: one strip context per device
  swf_group* group_ = nullptr;
  double group_vol_[3] = {0.0, 0.0, 0.0};
  mutable TimestepControl pushed_ctl_;
  mutable StepperOptions pushed_opt_;
  // host caches for the accessors (filled from the device on demand)
  mutable BlockMask mask_;
  mutable SourceField src_;
  mutable ForceField f_n_, f_mid_;
  mutable std::vector<double> buf_[9];
};

}  // namespace swflood
