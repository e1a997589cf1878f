/*
 * swf.h — C ABI of the B200-native CSPH-TVD time step (libswflood_cuda.so).
 *
 * This is the drop-in boundary for the one hot path this repository builds:
 * swflood::CsphTvdStepper::step (reference: proj/src/stepper.cpp:706-749) and
 * the surrounding solver API of proj/include/swflood/stepper.hpp:76-169.
 * The reference has no FFI of its own; the entry points below
 * are the ones a binding for that C++ class needs, one per public member, with
 * plain pointers and sizes only.  Citations are relative to /root/reference.
 *
 * Status codes mirror the reference's error convention
 * (proj/include/swflood/errors.hpp:8-21, proj/src/grid.cpp:102-110):
 *   SWF_OK 0, SWF_ECONFIG 1 (ConfigError), SWF_ENUMERICAL 2 (NumericalError),
 *   SWF_ERANGE 3 (std::out_of_range), SWF_ECUDA 4 (device/runtime failure).
 * The message text of the last failure is returned by swf_last_error(ctx)
 * (ctx may be NULL for failures of swf_create).  On SWF_ENUMERICAL the flow
 * state is left exactly as it was before the failing step, like the
 * reference, which throws before FlowState is modified.
 *
 * Threading: one host thread per swf_ctx, like the reference's externally
 * single-stepped stepper.  Every context owns one CUDA stream.
 */
#ifndef SWF_H_
#define SWF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWF_OK 0
#define SWF_ECONFIG 1
#define SWF_ENUMERICAL 2
#define SWF_ERANGE 3
#define SWF_ECUDA 4

/* EdgeKind, stepper.hpp:20 */
#define SWF_EDGE_REFLECTIVE 0
#define SWF_EDGE_OPEN 1

/* SourceSpec::Kind, sources.hpp:25-26 */
#define SWF_SOURCE_DISCHARGE 0
#define SWF_SOURCE_RAIN 1

/* Terrain, grid.hpp:18-37.  b is row-major, k = i + j*nx, j northward. */
typedef struct swf_terrain {
  int nx, ny;
  double h;
  double x0, y0;
  const double* b; /* nx*ny host doubles, copied to the device at creation */
} swf_terrain;

/* PhysicalParams, grid.hpp:59-74 (defaults grid.hpp:60-68). */
typedef struct swf_params {
  double g, n_manning, nu, omega_z, c_a, rho_air, rho_water, eps_dry;
  const double* n_field; /* NULL = scalar n_manning; else nx*ny host doubles */
} swf_params;

/* TimestepControl, stepper.hpp:13-18 */
typedef struct swf_control {
  double courant, dt_max, dt_min;
} swf_control;

/* StepperOptions + BoundaryConfig, stepper.hpp:22-28,59-64.
 * `workers` is accepted and ignored on the GPU. */
typedef struct swf_options {
  int block_size;
  int skip_dry_blocks;
  int workers;
  int west, east, south, north; /* SWF_EDGE_* */
} swf_options;

/* SourceSpec, sources.hpp:25-36 (name omitted; rect is inclusive). */
typedef struct swf_source {
  int kind; /* SWF_SOURCE_* */
  int i0, j0, i1, j1;
  int n_hydro;
  const double* hydro_t; /* n_hydro strictly increasing times */
  const double* hydro_q; /* n_hydro discharges [m^3/s] */
  double rate;           /* rain sigma [m/s] */
  double vx, vy;         /* source water velocity */
} swf_source;

/* StepInfo + StageTimings, stepper.hpp:31-57.  timings[] are seconds of
 * device time per stage bucket (mask, forces, dt, predictor, mid_forces,
 * corrector, flux, finalize) when timing is enabled, else zeros. */
typedef struct swf_step_info {
  double tau;
  double active_fraction;
  int lagrangian_blocks, flux_blocks, total_blocks;
  double timings[8];
  double clamp_deficit_volume;
  double source_volume;
  double boundary_outflow_volume;
} swf_step_info;

/* Stage ids for swf_stage, stepper.hpp:88-96 (step() composes these). */
enum swf_stage_id {
  SWF_STAGE_BEGIN = 0,       /* begin_step      stepper.cpp:172-201 */
  SWF_STAGE_FORCES = 1,      /* compute_forces  stepper.cpp:210-222 */
  SWF_STAGE_DT = 2,          /* compute_dt      stepper.cpp:224-267 */
  SWF_STAGE_PREDICTOR = 3,   /* predictor       stepper.cpp:269-308 */
  SWF_STAGE_MID_FORCES = 4,  /* mid_forces      stepper.cpp:310-333 */
  SWF_STAGE_CORRECTOR = 5,   /* corrector       stepper.cpp:335-400 */
  SWF_STAGE_FLUX = 6,        /* flux            stepper.cpp:579-626 */
  SWF_STAGE_FINAL = 7        /* final_update    stepper.cpp:628-704 */
};

/* Scratch ids for swf_download_scratch, the span accessors of
 * stepper.hpp:103-119. */
enum swf_scratch_id {
  SWF_SCR_FN_FX = 0, SWF_SCR_FN_FY, SWF_SCR_FN_FRIC_X, SWF_SCR_FN_FRIC_Y,
  SWF_SCR_FN_SIGMA,                                   /* forces_n()   */
  SWF_SCR_FM_FX, SWF_SCR_FM_FY, SWF_SCR_FM_FRIC_X, SWF_SCR_FM_FRIC_Y,
  SWF_SCR_FM_SIGMA,                                   /* forces_mid() */
  SWF_SCR_HALF_H, SWF_SCR_HALF_HUX, SWF_SCR_HALF_HUY, /* half_depth() + momenta */
  SWF_SCR_HT, SWF_SCR_HVTX, SWF_SCR_HVTY,             /* lagrangian_*()  */
  SWF_SCR_DRX, SWF_SCR_DRY,                           /* displacement_*() */
  SWF_SCR_FH, SWF_SCR_FVX, SWF_SCR_FVY,               /* flux_*()     */
  SWF_SCR_SIGMA, SWF_SCR_SRC_VX, SWF_SCR_SRC_VY,      /* step_sources() */
  SWF_SCR_COUNT
};

typedef struct swf_ctx swf_ctx;

/* ---- lifecycle: CsphTvdStepper::CsphTvdStepper, stepper.cpp:127-159 ---- */
int swf_create(const swf_terrain* terrain, const swf_params* params,
               const swf_control* control, const swf_options* options,
               swf_ctx** out);
void swf_destroy(swf_ctx* ctx);
const char* swf_last_error(const swf_ctx* ctx);

/* ---- configuration: set_wind / set_sources, stepper.cpp:161-170;
 *      control() / options() mutable accessors, stepper.hpp:100-101 ---- */
int swf_set_wind(swf_ctx* ctx, int n, const double* t, const double* wx,
                 const double* wy);
int swf_set_sources(swf_ctx* ctx, int n, const swf_source* sources);
int swf_set_control(swf_ctx* ctx, const swf_control* control);
int swf_get_control(const swf_ctx* ctx, swf_control* control);
int swf_set_options(swf_ctx* ctx, const swf_options* options);
int swf_get_options(const swf_ctx* ctx, swf_options* options);

/* ---- state: FlowState, grid.hpp:42-57.  Host arrays of nx*ny doubles. ---- */
int swf_upload_state(swf_ctx* ctx, const double* H, const double* HUx,
                     const double* HUy, double t);
int swf_download_state(swf_ctx* ctx, double* H, double* HUx, double* HUy,
                       double* t);
/* Device pointers of the resident state (zero-copy interop).  They change
 * after every successful step (ping-pong buffers). */
int swf_device_state(swf_ctx* ctx, double** H, double** HUx, double** HUy);

/* ---- the hot path: CsphTvdStepper::step, stepper.cpp:706-749 ---- */
/* Drop-in form of step(FlowState&, dt_cap): host buffers in, host buffers
 * out, t advanced in place. */
int swf_step_host(swf_ctx* ctx, double* H, double* HUx, double* HUy,
                  double* t, double dt_cap, swf_step_info* info);
/* Host bytes the last swf_step_host read: with PINNED (device-mapped) arrays
 * the depth in full plus the momentum of the flux-active tiles only (sparse
 * zero-copy ingest; afterwards the resident calls need swf_upload_state);
 * otherwise the three full fields. */
int swf_last_ingest_bytes(const swf_ctx* ctx, long long* bytes);
/* Host bytes the last synchronised pinned host-buffer step wrote back (the
 * updated cells of its flux-on blocks, counted on the device). */
int swf_last_writeback_bytes(swf_ctx* ctx, long long* bytes);
/* Opt-in host mirror for swf_step_host on PINNED arrays (SURVEY.md §8b,
 * "Ownership"; off by default).  On: after a host step the device keeps
 * the state it wrote into the caller's arrays, and the next host step with
 * the SAME arrays and the t it returned skips every host->device copy (the
 * first step, other arrays, another t, or any resident/upload/stage call in
 * between make it upload the three fields in full once).  The caller
 * promises not to change the arrays between host steps, or declares a
 * change with swf_host_changed(ctx).  Results are identical either way. */
int swf_set_host_mirror(swf_ctx* ctx, int on);
/* "exact" (libswflood_cuda.so: bit-identical to the reference, -fmad=false)
 * or "fast" (libswflood_cuda_fast.so, opt-in: FMA contraction, CUDA cbrt,
 * reciprocal multiplications; validated to a stated tolerance with tau
 * pinned, the wet/dry mask bit-exact -- tests/test_gpu_fast.py). */
const char* swf_build_flavor(void);
int swf_host_changed(swf_ctx* ctx);
/* Tiles of the last synchronised step whose speculative divisions were
 * rejected and that were recomputed exactly: counts[0] forces, [1] step
 * (diagnostics; see the speculative-division note in swf_fused.cu). */
int swf_debug_redo_counts(const swf_ctx* ctx, int* counts);
/* How k_step stages its tile regions: 1 = TMA tensor copies
 * (cp.async.bulk.tensor; needs an even nx), 0 = per-thread loads.  Results
 * are identical either way (diagnostics). */
int swf_debug_region_loads(const swf_ctx* ctx);
/* One step on the device-resident state; info may be NULL (then no host
 * synchronisation happens and errors surface at the next synchronising
 * call). */
int swf_step(swf_ctx* ctx, double dt_cap, swf_step_info* info);
/* n steps on the device-resident state without host synchronisation in
 * between (CUDA-graph replay).  Stops at the first failing step, leaving the
 * state as it was before that step; *done receives the steps completed. */
int swf_run(swf_ctx* ctx, int n, double dt_cap, int* done,
            swf_step_info* last);
/* Tiles (32 x 16 cells) the last fused step updated; swf_step_host writes
 * back only these when the host arrays are pinned (the rest kept their
 * step-start values, which the caller's arrays already hold). */
int swf_active_tiles(swf_ctx* ctx, int* n_active, int* n_total,
                     int* cells_per_tile);
/* Synchronise the context's stream and report a pending device error. */
int swf_sync(swf_ctx* ctx);
/* Device timing with CUDA events on the context's stream.  slots == 0: off;
 * 1: swf_step_info.timings of the last step; > 1: a ring of `slots` per-step
 * event sets readable with swf_timing_read (swf_run then launches directly
 * instead of replaying its CUDA graph).  Fused-path buckets: mask = begin +
 * K1, forces = K2+K3 kernel, dt = tau kernel, flux = fused K4..K8 kernel,
 * finalize = diagnostics/commit; predictor/mid_forces/corrector are 0. */
int swf_set_timing(swf_ctx* ctx, int slots);
/* Per-step bucket seconds of the last nsteps fused steps: out[nsteps*8]. */
int swf_timing_read(swf_ctx* ctx, int nsteps, double* out);
/* The CUDA stream (cudaStream_t) of the context, for interop. */
void* swf_stream(swf_ctx* ctx);
/* Execution path of swf_step / swf_run: 0 = fused tile kernels (default),
 * 1 = the unfused stage kernels (one per reference stage; keeps every
 * scratch accessor current, like the reference). */
int swf_set_mode(swf_ctx* ctx, int mode);

/* ---- stage API (stepper.hpp:88-96) for stage-differential tests. ---- */
/* arg is dt_cap for SWF_STAGE_DT and tau for the later stages; the tau that
 * SWF_STAGE_DT computes is written to *tau_out (may be NULL). */
int swf_stage(swf_ctx* ctx, int stage, double arg, double* tau_out);
/* Span accessors (stepper.hpp:103-119): nx*ny doubles. */
int swf_download_scratch(swf_ctx* ctx, int which, double* out);
/* BlockMask counts (block.hpp:20-36), total_blocks ints each; nbx/nby out. */
int swf_download_mask(swf_ctx* ctx, int* interior, int* halo, int* nbx,
                      int* nby);
/* last_clamp_deficit / last_source_volume / last_boundary_outflow,
 * stepper.hpp:117-119. */
int swf_last_volumes(swf_ctx* ctx, double* clamp_deficit, double* source_volume,
                     double* boundary_outflow);

/* ---- free per-cell functions evaluated ON THE DEVICE (KAT tests) ---- */
/* hll_face_flux, riemann.hpp:18-19: in = n x {hL,unL,utL,hR,unR,utR},
 * out = n x {fm,fn,ft}. */
int swf_dev_hll_face_flux(int n, const double* in, double g, double* out);
/* the shared-reciprocal division of the kernels against plain IEEE division:
 * in = n x {a, b}, out = n x {rdiv(a, recip_of(b)), a/b} (must be equal). */
int swf_dev_rdiv(int n, const double* ab, double* out);
/* the speculative form the fused kernels use: out = n x {q, accepted}; an
 * accepted q must equal a/b bit for bit (rejected items are redone exactly). */
int swf_dev_rdiv_spec(int n, const double* ab, double* out);
/* the square root of the fused kernels: out = n x {q, accepted}; an accepted
 * q must equal the IEEE sqrt(x) bit for bit (the fast path without its slow
 * branch when built with SWF_SPEC_SQRT, else sqrt itself, always accepted). */
int swf_dev_sqrt_spec(int n, const double* x, double* out);
/* the libm-compatible cube root used by friction (forcing.hpp:81). */
int swf_dev_cbrt(int n, const double* x, double* y);
/* bottom_friction, forcing.cpp:26-28: in = n x {ux,uy,H}, out = n x {fx,fy}. */
int swf_dev_bottom_friction(int n, const double* in, double g, double n_manning,
                            double* out);
/* assemble_forces, forcing.hpp:51-54 (forcing.cpp:58-70): the ForceField of
 * every cell of the state (H, HUx, HUy: nx*ny host doubles).  The wind is
 * already sampled at t (WindForcing::at, host); has_wind = wind.any().
 * sigma/svx/svy: the SourceField (NULL sigma = empty field).  Any output may
 * be NULL.  terrain->b and params->n_field as for swf_create. */
int swf_dev_assemble_forces(const swf_terrain* terrain, const swf_params* params,
                            const double* H, const double* HUx, const double* HUy,
                            int has_wind, double wx, double wy, const double* sigma,
                            const double* svx, const double* svy, double* fx, double* fy,
                            double* fric_x, double* fric_y, double* sigma_eff);
/* viscous_force (forcing.hpp:34-35, which = 0) and surface_gradient_force
 * (forcing.hpp:46-47, which = 1) at npt cells ij = npt x {i, j}:
 * out = npt x {fx, fy}.  SWF_ERANGE for a cell outside the grid. */
#define SWF_POINT_VISCOUS 0
#define SWF_POINT_SURFACE_GRADIENT 1
int swf_dev_point_forces(const swf_terrain* terrain, const swf_params* params,
                         const double* H, const double* HUx, const double* HUy, int which,
                         int npt, const int* ij, double* out);
/* coriolis_force, forcing.hpp:38: u = n x {ux, uy}, out = n x {fx, fy}. */
int swf_dev_coriolis_force(int n, const double* u, double omega_z, double* out);
/* wind_force, forcing.hpp:42-43, with W = wind.at(t) sampled by the caller:
 * in = n x {ux, uy, H}, out = n x {fx, fy} (c_a, rho_air, rho_water from params). */
int swf_dev_wind_force(int n, const double* in, double wx, double wy,
                       const swf_params* params, double* out);
/* compute_block_mask, block.hpp:38-39: interior/halo = nbx*nby ints with
 * nbx = ceil(nx/B), nby = ceil(ny/B); index_q may be NULL (no sources). */
int swf_dev_block_mask(int nx, int ny, const double* H, const uint8_t* index_q,
                       double eps_dry, int block_size, int* interior, int* halo);
/* source_terms (sources.hpp:40-41, resample = 0: fills sigma, vx, vy and
 * index_q) and resample_sigma (sources.hpp:45-46, resample = 1: sigma only;
 * vx, vy, index_q untouched and may be NULL), all nx*ny. */
int swf_dev_source_terms(const swf_terrain* terrain, const swf_source* sources, int n_sources,
                         double t, int resample, double* sigma, double* vx, double* vy,
                         uint8_t* index_q);

/* ---- row-strip decomposition (multi-GPU) ---- */
/* A strip context owns global rows [j0, j1) of an nx x ny_global domain and
 * keeps SWF_HALO ghost rows on each interior side.  terrain->ny must equal
 * ny_global; terrain->b and params->n_field point at the strip's window, the
 * global rows [j0 - ghosts, j1 + ghosts) (swf_strip_rows reports the ghost
 * counts).  device selects the CUDA device. */
#define SWF_HALO 3
int swf_create_strip(const swf_terrain* terrain, const swf_params* params,
                     const swf_control* control, const swf_options* options,
                     int j0, int j1, int device, swf_ctx** out);
/* Split step for strips.  Before phase 1 the caller fills the ghost rows of
 * the current state (swf_strip_halo_ptrs).  Phase 1 computes sources, the
 * block mask and the forces, and returns this strip's CFL speed (an exact,
 * non-negative double; synchronises the stream).  Phase 2 takes the global
 * max speed over all strips (an exact allreduce-max), computes tau and
 * finishes the step; info (may be NULL) reports this strip's blocks. */
int swf_strip_phase1(swf_ctx* ctx, double dt_cap, double* speed_out);
int swf_strip_phase2(swf_ctx* ctx, double global_speed, double dt_cap,
                     swf_step_info* info);
/* Device addresses of the halo rows of the CURRENT state for the exchange:
 * side 0 = south (lower j), 1 = north.  send3/recv3 receive the H, HUx, HUy
 * pointers of the SWF_HALO owned boundary rows and of the ghost rows;
 * *count = doubles per field (0 when that side is a domain edge). */
int swf_strip_halo_ptrs(swf_ctx* ctx, int side, double** send3, double** recv3,
                        size_t* count);
/* Copy the SWF_HALO owned boundary rows of `side` into the contiguous DEVICE
 * buffer dst = [H | HUx | HUy] (3*count doubles), or a neighbour's pack into
 * this strip's ghost rows on `side`.  Synchronous on the context stream. */
int swf_strip_pack(swf_ctx* ctx, int side, double* dst);
int swf_strip_unpack(swf_ctx* ctx, int side, const double* src);
/* Asynchronous strip steps (no host synchronisation inside a batch, so the
 * halo exchange and the dt allreduce can run as device-side collectives on
 * the context stream, overlapped with interior compute):
 *   swf_strip_begin_batch(ctx)
 *   per step:  pack_async(side) -> exchange starts on the comm stream
 *              swf_strip_forces(ctx, dt_cap, 0)   begin + interior tile rows
 *              (exchange done) unpack_async(side)
 *              swf_strip_forces(ctx, dt_cap, 1)   ghost-dependent tile rows
 *              (block sizes not dividing 16: part 0 is empty and part 1
 *               runs the whole phase 1 -- same results, no overlap)
 *              swf_strip_local_speed(ctx, dev)    strip CFL speed -> device
 *              (allreduce-MAX of dev across strips, on the device, over the
 *               8 bytes as int64: a stopped strip publishes a marker above
 *               every speed, and every strip's finish then stops as well)
 *              swf_strip_finish(ctx, dev, dt_cap) tau from *dev, K4..K8
 *   swf_strip_end_batch(ctx, &done, &last)        sync + commit (like swf_run)
 *   (allreduce-MIN of done across strips)
 *   swf_strip_settle(ctx, ok)                     commit ok = min(done) steps
 * A strip that aborts in step k stops the others in step k + 1 (before their
 * K4..K8), so every strip has done ok or ok + 1 steps and settle rolls the
 * latter back by one (the other ping-pong buffer, the previous t).  A strip
 * stopped only by that marker reports SWF_ENUMERICAL "strip stopped: ...".
 * Every call is enqueued on the context stream (swf_stream). */
int swf_strip_begin_batch(swf_ctx* ctx);
int swf_strip_forces(swf_ctx* ctx, double dt_cap, int part);
int swf_strip_local_speed(swf_ctx* ctx, double* dev_out);
int swf_strip_finish(swf_ctx* ctx, const double* dev_global_speed, double dt_cap);
int swf_strip_end_batch(swf_ctx* ctx, int* done, swf_step_info* last);
int swf_strip_settle(swf_ctx* ctx, int ok);
/* steps the last batch committed on this strip (after swf_strip_end_batch,
 * also when it returned an error) */
int swf_strip_steps_done(const swf_ctx* ctx);
int swf_strip_pack_async(swf_ctx* ctx, int side, double* dst);
int swf_strip_unpack_async(swf_ctx* ctx, int side, const double* src);
/* P2P halo (fused exchange): the base pointers of this context's six state
 * buffers [H0, H1, HUx0, HUx1, HUy0, HUy1] (for cudaIpcGetMemHandle), and
 * registration of a neighbour's six buffers mapped into this process (side 0 =
 * south neighbour, 1 = north; peer_row0 = the global row of the neighbour's
 * local row 0; bufs6 = NULL unregisters).  With a peer registered, k_step
 * stores every owned cell within SWF_HALO rows of that strip edge also into
 * the neighbour's ghost rows of the next-parity buffer and fences, so the
 * exchange reduces to a stream-ordered token per step (multigpu.py). */
int swf_device_buffers(swf_ctx* ctx, double** out6);
int swf_strip_set_peer(swf_ctx* ctx, int side, double* const* bufs6, int peer_row0);
/* Owned global rows [j0, j1) and the ghost-row counts below/above. */
int swf_strip_rows(const swf_ctx* ctx, int* j0, int* j1, int* ghost_lo,
                   int* ghost_hi);

/* Host-buffer step of a strip from PINNED window arrays (rows = its window,
 * the caller's own layout): phase 1 copies the depth window, computes the
 * block mask, reads the momentum of the flux-active owned tiles and of every
 * ghost row over PCIe, runs the forces and returns the strip's CFL speed;
 * the caller max-reduces it over the strips; phase 2 finishes the step with
 * the global speed, k_step writing every updated owned cell straight into the
 * caller's arrays (restored on a numerical abort); *t = the new time.  The
 * device copy is incomplete afterwards (upload before resident steps). */
int swf_strip_host_phase1(swf_ctx* ctx, double* H, double* HUx, double* HUy, const double* t,
                          double dt_cap, double* speed_out);
int swf_strip_host_phase2(swf_ctx* ctx, double* H, double* HUx, double* HUy, double* t,
                          double global_speed, double dt_cap, swf_step_info* info);

/* ---- single-process multi-GPU group (StepperOptions::devices > 1) ----
 * Replaces CsphTvdStepper's internal one-stream-per-GPU model of SURVEY.md
 * §8b for callers that drive every GPU from one process: n strip contexts
 * (swf_create_strip, ascending adjacent rows, each on its own device, devices
 * may repeat).  The group enables peer access, links neighbours so every
 * k_step stores its boundary rows into the neighbours' ghost rows, orders the
 * devices' streams with events (no host synchronisation inside a run) and
 * max-reduces the CFL speed on the first strip's device.  The strips' ghost
 * rows must be current when a run starts (upload whole windows).  All strips
 * commit the same number of steps (the fewest any completed); info = the
 * group's last step (block counts and volumes summed over the strips). */
typedef struct swf_group swf_group;
int swf_group_create(swf_ctx* const* strips, int n, swf_group** out);
int swf_group_run(swf_group* g, int nsteps, double dt_cap, int* done, swf_step_info* last);
const char* swf_group_last_error(const swf_group* g);
void swf_group_destroy(swf_group* g);
/* number of CUDA devices visible to the process */
int swf_device_count(int* n);

/* ---- two-level nested grids (SPEC.md [MODULE] nesting) ----
 * The reference ships no code for this module; these entry
 * points implement its SPEC operations prolong_boundary,
 * restrict_feedback (:379-385) and coupled_step (:386-392) on the device.
 * The operator details are in paper_1705_00614_b200/csrc/swf_nest.cu.
 * A nest couples a global (coarse) context with a fine context created for
 * the window at h/r plus a ghost band: fine nx = r*ni + 2*ghost, ny likewise,
 * fine h = coarse h / r, same device, not strip contexts. */
typedef struct swf_nest swf_nest;
typedef struct swf_nest_desc {
  int i0, j0, ni, nj; /* window: coarse cells [i0, i0+ni) x [j0, j0+nj) */
  int r;              /* refinement factor (>= 1) */
  int ghost;          /* ghost band width in fine cells (SPEC default 2) */
  int two_way;        /* 1: restrict_feedback after each coupled step */
} swf_nest_desc;
typedef struct swf_coupled_info {
  double tau;           /* the global step's tau */
  int substeps_total;   /* fine steps over all nests */
  int substeps_max;     /* most fine steps of one nest */
  double fine_tau_min;  /* smallest fine tau */
  swf_step_info coarse; /* the global step */
  double reflux_clamp_volume; /* volume added where the flux correction would
                                 have emptied a dry-side cell (mass ledger) */
} swf_coupled_info;
int swf_nest_create(swf_ctx* coarse, swf_ctx* fine, const swf_nest_desc* desc,
                    swf_nest** out);
void swf_nest_destroy(swf_nest* nest);
const char* swf_nest_last_error(const swf_nest* nest);
/* ghost cells of the fine grid: nxf*nyf - (r*ni)*(r*nj) */
int swf_nest_ghost_count(const swf_nest* nest, size_t* count);
/* prolong_boundary of the coarse CURRENT state into ghost slot 0 or 1 */
int swf_nest_prolong(swf_nest* nest, int slot);
/* the fine ghost band := lerp(slot 0, slot 1, alpha) */
int swf_nest_apply_ghosts(swf_nest* nest, double alpha);
/* restrict_feedback: window cells := means of their r x r fine cells */
int swf_nest_restrict(swf_nest* nest);
/* slot values [H | HUx | HUy], 3*count doubles, ghost-cell order */
int swf_nest_download_ghosts(swf_nest* nest, int slot, double* out);
/* coupled_step: one global step (dt_cap as in step()), then every nest
 * subcycles to the new global time with time-interpolated ghosts and, when
 * two_way, restricts.  The fine contexts must be at the global time. */
int swf_coupled_step(swf_ctx* coarse, swf_nest** nests, int n_nests, double dt_cap,
                     swf_coupled_info* info);

#ifdef __cplusplus
}
#endif
#endif /* SWF_H_ */
