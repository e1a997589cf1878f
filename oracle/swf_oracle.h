/*
 * swf_oracle.h — TEST INFRASTRUCTURE ONLY.  The checker ABI shared by
 *   - liborc.so           (swf_oracle.c: a plain-C restatement of the
 *                          reference algorithm, in git), and
 *   - _ref/libswflood_ref.so (ref_harness.cpp: the real reference compiled
 *                          from /root/reference, git-ignored).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load either library.  The product path
 * (libswflood_cuda.so) never links or calls anything here.
 *
 * Struct types come from the public C ABI header so that both sides of a
 * parity test describe a case with the very same bytes.
 */
#ifndef SWF_ORACLE_H_
#define SWF_ORACLE_H_

#include "swf.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_ctx orc_ctx;

int orc_create(const swf_terrain* terrain, const swf_params* params,
               const swf_control* control, const swf_options* options,
               orc_ctx** out);
void orc_destroy(orc_ctx* ctx);
const char* orc_last_error(const orc_ctx* ctx);
int orc_set_wind(orc_ctx* ctx, int n, const double* t, const double* wx,
                 const double* wy);
int orc_set_sources(orc_ctx* ctx, int n, const swf_source* sources);
int orc_set_control(orc_ctx* ctx, const swf_control* control);
int orc_set_options(orc_ctx* ctx, const swf_options* options);
int orc_set_state(orc_ctx* ctx, const double* H, const double* HUx,
                  const double* HUy, double t);
int orc_get_state(orc_ctx* ctx, double* H, double* HUx, double* HUy, double* t);
int orc_step(orc_ctx* ctx, double dt_cap, swf_step_info* info);
int orc_run(orc_ctx* ctx, int n, double dt_cap, int* done, swf_step_info* last);
int orc_stage(orc_ctx* ctx, int stage, double arg, double* tau_out);
int orc_scratch(orc_ctx* ctx, int which, double* out);
int orc_mask(orc_ctx* ctx, int* interior, int* halo, int* nbx, int* nby);
int orc_face_fm(orc_ctx* ctx, int dir, double* out);
int orc_volumes(orc_ctx* ctx, double* clamp_deficit, double* source_volume,
                double* boundary_outflow);

/* free functions (forcing.hpp:29-57, riemann.hpp:18-19, grid.hpp:77,114-121) */
double orc_cbrt(double x);
void orc_hll_face_flux(const double* in6, double g, double* out3);
void orc_bottom_friction(double ux, double uy, double H, double g, double n,
                         double* out2);
void orc_coriolis_force(double ux, double uy, double omega_z, double* out2);
void orc_wind_force(double ux, double uy, double H, double wx, double wy,
                    double c_a, double rho_air, double rho_water, double* out2);
/* per-cell force terms on a full state (cell (i,j)); status like orc_* */
int orc_viscous_force(const swf_terrain* terrain, const swf_params* params,
                      const double* H, const double* HUx, const double* HUy,
                      int i, int j, double* out2);
int orc_surface_gradient_force(const swf_terrain* terrain,
                               const swf_params* params, const double* H,
                               const double* HUx, const double* HUy, int i,
                               int j, double* out2);
double orc_total_volume(int n, const double* H, double h);
double orc_latitude_to_omega_z(double latitude_deg);

#ifdef __cplusplus
}
#endif
#endif /* SWF_ORACLE_H_ */
