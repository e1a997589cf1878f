// swflood/io.hpp — scenario I/O (SPEC.md [MODULE] scenario_io):
// the on-disk formats that feed terrain and state to the step and carry its
// results out.  SPEC-only in the reference (no header ships), so the names
// follow the SPEC operations: load_terrain (:436-443), load_scenario
// (:444-451), write_snapshot (:452-458).  Host code (parsing, formatting);
// nothing here is on the per-cell path.
#pragma once

#include <cstdio>
#include <span>
#include <string>
#include <vector>

#include "../swflood_b200.hpp"

namespace swflood::io {

// Impermeable high ground for NODATA cells.
constexpr double kNoDataBed = 1.0e4;

// ESRI ASCII grid: ncols, nrows, xllcorner|xllcenter, yllcorner|yllcenter,
// cellsize, optional NODATA_value; then nrows rows NORTH to SOUTH.  The
// Terrain is row-major with j increasing northward (grid.hpp:15-17), so file
// row r is j = nrows - 1 - r.  Errors: ConfigError naming the line.
Terrain load_terrain(const std::string& path);

// A raster in the same format (round-trips through load_raster/load_terrain),
// values printed with %.6e unless `precision` says otherwise.
void write_raster(const std::string& path, int nx, int ny, double x0, double y0, double h,
                  std::span<const double> values, double nodata = -9999.0, int precision = 6);
// Values of a raster (NODATA cells -> `nodata_as`), same orientation rules.
std::vector<double> load_raster(const std::string& path, int* nx, int* ny, double* h = nullptr,
                                double* x0 = nullptr, double* y0 = nullptr,
                                double nodata_as = kNoDataBed);

// ScenarioConfig: a key = value file with [sections]
// (grammar in DESIGN.md §8); relative paths resolve against its directory.
struct ScenarioConfig {
  std::string terrain_path;   // ESRI ASCII DEM (or empty with synthetic)
  std::string synthetic;      // "floodplain N H" / "lake N H LEVEL" / "dam N" (built-in)
  PhysicalParams params;
  TimestepControl control;
  StepperOptions options;
  std::vector<SourceSpec> sources;
  WindForcing wind;
  std::string initial = "dry";  // dry | level | raster
  double initial_level = 0.0;
  std::string initial_raster;
  double duration = 0.0;
  double cadence = 0.0;
  unsigned seed = 1705;
};

ScenarioConfig load_scenario(const std::string& path);
// The terrain the config names (loaded or generated) and its initial state.
Terrain scenario_terrain(const ScenarioConfig& cfg);
FlowState scenario_initial_state(const ScenarioConfig& cfg, const Terrain& terrain);

// Snapshot rasters H, Ux, Uy, eta at time t into dir/<stem>_{H,Ux,Uy,eta}.asc
// (SPEC.md:452-458); velocities are 0 where H <= eps_dry.
void write_snapshot(const FlowState& state, const Terrain& terrain, const PhysicalParams& params,
                    const std::string& dir, const std::string& stem);

// Summary CSV: t, total volume, wet fraction, max |U|, tau (one row per
// snapshot plus the mass-balance ledger columns).
struct SummaryRow {
  double t = 0.0, volume = 0.0, wet_fraction = 0.0, max_speed = 0.0, tau = 0.0;
  double source_volume = 0.0, outflow_volume = 0.0, clamp_deficit = 0.0;
  long steps = 0;
};
SummaryRow summarize(const FlowState& state, const Terrain& terrain, const PhysicalParams& params);
class SummaryWriter {
 public:
  explicit SummaryWriter(const std::string& path);
  ~SummaryWriter();
  void row(const SummaryRow& r);
  int rows() const { return rows_; }

 private:
  std::FILE* f_ = nullptr;
  int rows_ = 0;
};

}  // namespace swflood::io
