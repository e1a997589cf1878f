// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.  Exposes the REAL reference
// (swflood::CsphTvdStepper, /root/reference/proj) through the checker ABI of
// swf_oracle.h so the Python tests and the CPU-baseline leg of bench.py can
// drive it.  Built by oracle/Makefile into oracle/_ref/libswflood_ref.so.
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "swflood/errors.hpp"
#include "swflood/forcing.hpp"
#include "swflood/grid.hpp"
#include "swflood/riemann.hpp"
#include "swflood/sources.hpp"
#include "swflood/stepper.hpp"

#include "../oracle/swf_oracle.h"

using namespace swflood;

struct orc_ctx {
  Terrain terrain;
  FlowState state;
  std::unique_ptr<CsphTvdStepper> stepper;
  std::string err;
  double last_tau = 0.0;
};

namespace {

std::string g_err;

template <class F>
int guarded(orc_ctx* c, F&& f) {
  try {
    f();
    return SWF_OK;
  } catch (const ConfigError& e) {
    (c ? c->err : g_err) = e.what();
    return SWF_ECONFIG;
  } catch (const NumericalError& e) {
    (c ? c->err : g_err) = e.what();
    return SWF_ENUMERICAL;
  } catch (const std::out_of_range& e) {
    (c ? c->err : g_err) = e.what();
    return SWF_ERANGE;
  } catch (const std::exception& e) {
    (c ? c->err : g_err) = e.what();
    return SWF_ECUDA;
  }
}

Terrain make_terrain(const swf_terrain* t) {
  Terrain T;
  T.nx = t->nx;
  T.ny = t->ny;
  T.h = t->h;
  T.x0 = t->x0;
  T.y0 = t->y0;
  if (t->nx > 0 && t->ny > 0 && t->b)
    T.b.assign(t->b, t->b + static_cast<std::size_t>(t->nx) * t->ny);
  return T;
}

PhysicalParams make_params(const swf_params* p, std::size_t n) {
  PhysicalParams P;
  P.g = p->g;
  P.n_manning = p->n_manning;
  if (p->n_field) P.n_field.assign(p->n_field, p->n_field + n);
  P.nu = p->nu;
  P.omega_z = p->omega_z;
  P.c_a = p->c_a;
  P.rho_air = p->rho_air;
  P.rho_water = p->rho_water;
  P.eps_dry = p->eps_dry;
  return P;
}

StepperOptions make_options(const swf_options* o) {
  StepperOptions O;
  O.block_size = o->block_size;
  O.skip_dry_blocks = o->skip_dry_blocks != 0;
  O.workers = o->workers;
  auto ek = [](int v) { return v == SWF_EDGE_OPEN ? EdgeKind::Open : EdgeKind::Reflective; };
  O.boundaries = {ek(o->west), ek(o->east), ek(o->south), ek(o->north)};
  return O;
}

void fill_info(const StepInfo& s, swf_step_info* info) {
  if (!info) return;
  info->tau = s.tau;
  info->active_fraction = s.active_fraction;
  info->lagrangian_blocks = s.lagrangian_blocks;
  info->flux_blocks = s.flux_blocks;
  info->total_blocks = s.total_blocks;
  const StageTimings& t = s.timings;
  double v[8] = {t.mask, t.forces, t.dt, t.predictor, t.mid_forces, t.corrector, t.flux, t.finalize};
  std::memcpy(info->timings, v, sizeof v);
  info->clamp_deficit_volume = s.clamp_deficit_volume;
  info->source_volume = s.source_volume;
  info->boundary_outflow_volume = s.boundary_outflow_volume;
}

void copy_span(std::span<const double> s, double* out) {
  std::memcpy(out, s.data(), s.size() * sizeof(double));
}

void copy_vec(const std::vector<double>& s, double* out) {
  std::memcpy(out, s.data(), s.size() * sizeof(double));
}

}  // namespace

extern "C" {

int orc_create(const swf_terrain* terrain, const swf_params* params,
               const swf_control* control, const swf_options* options,
               orc_ctx** out) {
  *out = nullptr;
  auto c = std::make_unique<orc_ctx>();
  int rc = guarded(nullptr, [&] {
    c->terrain = make_terrain(terrain);
    TimestepControl C{control->courant, control->dt_max, control->dt_min};
    c->stepper = std::make_unique<CsphTvdStepper>(
        c->terrain, make_params(params, c->terrain.cells()), C, make_options(options));
    c->state = FlowState::dry(c->terrain);
  });
  if (rc == SWF_OK) *out = c.release();
  return rc;
}

void orc_destroy(orc_ctx* c) { delete c; }

const char* orc_last_error(const orc_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

int orc_set_wind(orc_ctx* c, int n, const double* t, const double* wx, const double* wy) {
  return guarded(c, [&] {
    WindForcing w;
    for (int k = 0; k < n; ++k) w.series.push_back({t[k], wx[k], wy[k]});
    c->stepper->set_wind(std::move(w));
  });
}

int orc_set_sources(orc_ctx* c, int n, const swf_source* s) {
  return guarded(c, [&] {
    std::vector<SourceSpec> v;
    for (int k = 0; k < n; ++k) {
      SourceSpec sp;
      sp.kind = s[k].kind == SWF_SOURCE_RAIN ? SourceSpec::Kind::Rain : SourceSpec::Kind::Discharge;
      sp.name = "src" + std::to_string(k);
      sp.cells = {s[k].i0, s[k].j0, s[k].i1, s[k].j1};
      for (int m = 0; m < s[k].n_hydro; ++m)
        sp.hydrograph.push_back({s[k].hydro_t[m], s[k].hydro_q[m]});
      sp.rate = s[k].rate;
      sp.source_velocity = {s[k].vx, s[k].vy};
      v.push_back(std::move(sp));
    }
    c->stepper->set_sources(std::move(v));
  });
}

int orc_set_control(orc_ctx* c, const swf_control* ctl) {
  return guarded(c, [&] {
    TimestepControl C{ctl->courant, ctl->dt_max, ctl->dt_min};
    c->stepper->control() = C;
  });
}

int orc_set_options(orc_ctx* c, const swf_options* o) {
  return guarded(c, [&] { c->stepper->options() = make_options(o); });
}

int orc_set_state(orc_ctx* c, const double* H, const double* HUx, const double* HUy, double t) {
  return guarded(c, [&] {
    std::size_t n = c->terrain.cells();
    c->state.H.assign(H, H + n);
    c->state.HUx.assign(HUx, HUx + n);
    c->state.HUy.assign(HUy, HUy + n);
    c->state.t = t;
  });
}

int orc_get_state(orc_ctx* c, double* H, double* HUx, double* HUy, double* t) {
  copy_vec(c->state.H, H);
  copy_vec(c->state.HUx, HUx);
  copy_vec(c->state.HUy, HUy);
  if (t) *t = c->state.t;
  return SWF_OK;
}

int orc_step(orc_ctx* c, double dt_cap, swf_step_info* info) {
  return guarded(c, [&] {
    StepInfo s = c->stepper->step(c->state, dt_cap);
    fill_info(s, info);
  });
}

int orc_run(orc_ctx* c, int n, double dt_cap, int* done, swf_step_info* last) {
  if (done) *done = 0;
  for (int k = 0; k < n; ++k) {
    int rc = orc_step(c, dt_cap, last);
    if (rc != SWF_OK) return rc;
    if (done) *done = k + 1;
  }
  return SWF_OK;
}

int orc_stage(orc_ctx* c, int stage, double arg, double* tau_out) {
  return guarded(c, [&] {
    CsphTvdStepper& s = *c->stepper;
    switch (stage) {
      case SWF_STAGE_BEGIN: s.begin_step(c->state); break;
      case SWF_STAGE_FORCES: s.compute_forces(c->state); break;
      case SWF_STAGE_DT: {
        double tau = s.compute_dt(c->state, arg);
        if (tau_out) *tau_out = tau;
        break;
      }
      case SWF_STAGE_PREDICTOR: s.predictor(c->state, arg); break;
      case SWF_STAGE_MID_FORCES: s.mid_forces(c->state, arg); break;
      case SWF_STAGE_CORRECTOR: s.corrector(c->state, arg); break;
      case SWF_STAGE_FLUX: s.flux(c->state, arg); break;
      case SWF_STAGE_FINAL: s.final_update(c->state, arg); break;
      default: throw ConfigError("unknown stage id");
    }
  });
}

int orc_scratch(orc_ctx* c, int which, double* out) {
  return guarded(c, [&] {
    CsphTvdStepper& s = *c->stepper;
    const ForceField& fn = s.forces_n();
    const ForceField& fm = s.forces_mid();
    switch (which) {
      case SWF_SCR_FN_FX: copy_vec(fn.fx, out); break;
      case SWF_SCR_FN_FY: copy_vec(fn.fy, out); break;
      case SWF_SCR_FN_FRIC_X: copy_vec(fn.fric_x, out); break;
      case SWF_SCR_FN_FRIC_Y: copy_vec(fn.fric_y, out); break;
      case SWF_SCR_FN_SIGMA: copy_vec(fn.sigma_eff, out); break;
      case SWF_SCR_FM_FX: copy_vec(fm.fx, out); break;
      case SWF_SCR_FM_FY: copy_vec(fm.fy, out); break;
      case SWF_SCR_FM_FRIC_X: copy_vec(fm.fric_x, out); break;
      case SWF_SCR_FM_FRIC_Y: copy_vec(fm.fric_y, out); break;
      case SWF_SCR_FM_SIGMA: copy_vec(fm.sigma_eff, out); break;
      case SWF_SCR_HALF_H: copy_span(s.half_depth(), out); break;
      case SWF_SCR_HT: copy_span(s.lagrangian_depth(), out); break;
      case SWF_SCR_HVTX: copy_span(s.lagrangian_momentum_x(), out); break;
      case SWF_SCR_HVTY: copy_span(s.lagrangian_momentum_y(), out); break;
      case SWF_SCR_DRX: copy_span(s.displacement_x(), out); break;
      case SWF_SCR_DRY: copy_span(s.displacement_y(), out); break;
      case SWF_SCR_FH: copy_span(s.flux_mass(), out); break;
      case SWF_SCR_FVX: copy_span(s.flux_momentum_x(), out); break;
      case SWF_SCR_FVY: copy_span(s.flux_momentum_y(), out); break;
      case SWF_SCR_SIGMA: copy_vec(s.step_sources().sigma, out); break;
      case SWF_SCR_SRC_VX: copy_vec(s.step_sources().vx, out); break;
      case SWF_SCR_SRC_VY: copy_vec(s.step_sources().vy, out); break;
      default: throw ConfigError("scratch not exposed by the reference API");
    }
  });
}

int orc_mask(orc_ctx* c, int* interior, int* halo, int* nbx, int* nby) {
  const BlockMask& m = c->stepper->mask();
  if (nbx) *nbx = m.nbx;
  if (nby) *nby = m.nby;
  if (interior) std::memcpy(interior, m.interior_wet.data(), m.interior_wet.size() * sizeof(int));
  if (halo) std::memcpy(halo, m.halo_wet.data(), m.halo_wet.size() * sizeof(int));
  return SWF_OK;
}

int orc_volumes(orc_ctx* c, double* cd, double* sv, double* bo) {
  if (cd) *cd = c->stepper->last_clamp_deficit();
  if (sv) *sv = c->stepper->last_source_volume();
  if (bo) *bo = c->stepper->last_boundary_outflow();
  return SWF_OK;
}

double orc_cbrt(double x) { return std::cbrt(x); }

void orc_hll_face_flux(const double* in, double g, double* out) {
  FaceFlux f = hll_face_flux(in[0], in[1], in[2], in[3], in[4], in[5], g);
  out[0] = f.fm;
  out[1] = f.fn;
  out[2] = f.ft;
}

void orc_bottom_friction(double ux, double uy, double H, double g, double n, double* out) {
  Vec2 f = bottom_friction({ux, uy}, H, g, n);
  out[0] = f.x;
  out[1] = f.y;
}

void orc_coriolis_force(double ux, double uy, double omega_z, double* out) {
  PhysicalParams p;
  p.omega_z = omega_z;
  Vec2 f = coriolis_force({ux, uy}, p);
  out[0] = f.x;
  out[1] = f.y;
}

void orc_wind_force(double ux, double uy, double H, double wx, double wy, double c_a,
                    double rho_air, double rho_water, double* out) {
  PhysicalParams p;
  p.c_a = c_a;
  p.rho_air = rho_air;
  p.rho_water = rho_water;
  Vec2 f = wind_force({ux, uy}, H, WindForcing::constant(wx, wy), 0.0, p);
  out[0] = f.x;
  out[1] = f.y;
}

static FlowState make_state(const swf_terrain* t, const double* H, const double* HUx,
                            const double* HUy) {
  FlowState s;
  s.nx = t->nx;
  s.ny = t->ny;
  std::size_t n = static_cast<std::size_t>(t->nx) * t->ny;
  s.H.assign(H, H + n);
  s.HUx.assign(HUx, HUx + n);
  s.HUy.assign(HUy, HUy + n);
  return s;
}

int orc_viscous_force(const swf_terrain* terrain, const swf_params* params, const double* H,
                      const double* HUx, const double* HUy, int i, int j, double* out) {
  return guarded(nullptr, [&] {
    Terrain T = make_terrain(terrain);
    FlowState s = make_state(terrain, H, HUx, HUy);
    Vec2 f = viscous_force(s, make_params(params, T.cells()), T, i, j);
    out[0] = f.x;
    out[1] = f.y;
  });
}

int orc_surface_gradient_force(const swf_terrain* terrain, const swf_params* params,
                               const double* H, const double* HUx, const double* HUy, int i,
                               int j, double* out) {
  return guarded(nullptr, [&] {
    Terrain T = make_terrain(terrain);
    FlowState s = make_state(terrain, H, HUx, HUy);
    Vec2 f = surface_gradient_force(s, T, make_params(params, T.cells()), i, j);
    out[0] = f.x;
    out[1] = f.y;
  });
}

double orc_total_volume(int n, const double* H, double h) {
  FlowState s;
  s.H.assign(H, H + n);
  Terrain T;
  T.h = h;
  return total_volume(s, T);
}

double orc_latitude_to_omega_z(double lat) { return latitude_to_omega_z(lat); }

}  // extern "C"
