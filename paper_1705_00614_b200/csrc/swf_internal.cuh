// swf_internal.cuh — device context of libswflood_cuda.so (not part of the ABI).
#pragma once

#include <cuda.h>  // CUtensorMap (TMA descriptors; encoded through the runtime's driver entry point)
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/swf.h"
#include "swf_math.cuh"

namespace swf {

// NVTX range over a host-side scope (SURVEY.md section 5 tracing): the
// stage buckets of a step (forces phase, k_step phase), host steps and runs
// show up by name in Nsight timelines.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// A source spec on the device (sources.hpp:25-36): rectangle, velocity, and
// the per-step sigma values at t_n and t_mid (computed by the begin/tau
// kernels, sources.cpp:37-41).
struct DevSrc {
  int kind, i0, j0, i1, j1, nh, off;  // off = offset into the hydrograph arrays
  double rate, vx, vy;
  double count_area;  // (double)count * (h*h), sources.cpp:40
};

constexpr int SPEED_SLOTS = 64;

// Device-resident per-step scalars.
struct StepScalars {
  double t;      // FlowState::t on the device
  double t_prev; // t before the last committed step (swf_strip_settle)
  double tau;    // this step's tau
  double t_mid;  // t + 0.5*tau
  double dt_cap;
  unsigned long long speed_bits;  // max CFL speed (non-negative double bits)
  unsigned long long speed_slots[SPEED_SLOTS];  // per-CTA maxima, spread
  double wind_n[2], wind_mid[2];
  unsigned long long err_key;  // (kind << 58) | detail; ~0ull = none
  double err_val[3];           // dt floor: cfl, dt_min, speed
  int lag_act, flux_act;  // active B-blocks (interior>0, interior|halo>0), owned
  int total_blocks;
  int steps_done;   // successful steps since the counter was reset
  int fail_step;    // step index of the first failure (-1 none)
  double deficit, srcvol, outflow;  // this step's diagnostics (volumes)
  double speed_local;               // strips: local max speed (phase 1 out)
  double dt_cap_dev;                // dt_cap of a step enqueued with dt_cap < 0 (k_tau)
  unsigned long long host_writes;   // doubles a host-buffer step wrote back (changed values only)
  int mask_valid;  // the tile flags of the previous step describe the current state
  int mask_fresh;  // != 0: k_mask/k_tiles just flagged the current state (host step);
                   // cleared by k_tau
  int redo_n[3];   // tiles queued for the exact redo: [0] k_forces, [1] k_step / k_flux, [2] k_lag
  int list_n[2];   // work-list lengths: [0] k_forces, [1] k_step (k_lag and k_flux share it)
  // k_step of this step may run (set by k_tau): an error raised BY this
  // step's k_step does not stop its other tiles or its redo tiles, so the
  // reported cell is the first in the reference's block order, not the
  // first found; an error from before (an earlier step, the dt floor, a
  // stopped peer strip, an idle substep) does
  int step_open;
  int list_take[3];  // work-list cursors of the persistent grids: [2] k_lag
};

// ERR_PEER: stopped because another strip of a swf_group aborted (ranks
// above every real error, so atomicMin keeps a strip's own error)
// ERR_IDLE: not an error -- a nested grid's device-driven subcycling reached
// the global time, so the remaining enqueued substeps of the batch skip
// (ranks above ERR_PEER; check_device_error reports it as success)
enum ErrKind : unsigned long long { ERR_DT = 1, ERR_CFL = 2, ERR_FLUX = 3, ERR_PEER = 7,
                                    ERR_IDLE = 8 };
constexpr unsigned long long ERR_NONE = ~0ull;
// A strip that has stopped publishes this as its CFL speed (the bits of a NaN
// above every non-negative double's bits): an int64 allreduce-MAX of the
// speeds then carries the stop to every rank, whose k_tau stops too.
constexpr unsigned long long SPEED_STOP_BITS = 0x7fffffffffffffffull;

// Every step kernel returns early once the context has stopped (an error,
// another strip's stop, or idle subcycling).
__device__ __forceinline__ bool stopped(const StepScalars* sc) { return sc->err_key != ERR_NONE; }

// Launch-invariant parameters of one context (passed by value to kernels).
struct Geo {
  int nx;        // columns
  int ny;        // GLOBAL rows
  int rows;      // local rows (owned + ghosts)
  int jg0;       // global row of local row 0
  int r0, r1;    // owned local rows [r0, r1)
  int bs, nbx, nby;     // B-blocks over the GLOBAL grid
  int bj0, bj1;         // owned block rows [bj0, bj1)
  int tiles_x, tiles_y; // fused-kernel tiles over owned rows
  int west_refl, east_refl, south_refl, north_refl;
  int skip;
  int has_nfield;
  int nsrc, nwind;
  double n_manning;
  double courant, dt_max, dt_min;
  PhysConst P;
};

// Face taps: the mass fluxes tau * fm through the faces on the boundary of a
// cell rectangle, recorded by k_step each step (nested-grid flux correction).
// Layout of a tap array: [west nj | east nj | south ni | north ni].
constexpr int MAX_TAPS = 4;
struct FaceTaps {
  int n = 0;
  int i0[MAX_TAPS], j0[MAX_TAPS], ni[MAX_TAPS], nj[MAX_TAPS];  // global cell rects
  double* out[MAX_TAPS];
};

struct Scratch;  // stage-path arrays (lazy)

}  // namespace swf

struct swf_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  swf::Geo geo{};
  double h = 0, x0 = 0, y0 = 0;
  swf_params params{};
  swf_control ctl{};
  swf_options opt{};
  // device arrays (local rows)
  double* b = nullptr;
  double* nf = nullptr;
  double* H[2] = {nullptr, nullptr};
  double* HUx[2] = {nullptr, nullptr};
  double* HUy[2] = {nullptr, nullptr};
  int cur = 0;
  double* fpx = nullptr;  // f_n.fx - f_n.fric_x (wet cells), fused path
  double* fpy = nullptr;
  double* d_lamn = nullptr;  // SWF_LAMBDA_SHARE builds: lambda(H_n, n) of the wet cells
  double* d_gxy = nullptr;   // SWF_GRAD_SHARE builds: k_step's half-step eta gradients
  // TMA descriptors of k_step's region loads: [parity][H, HUx, HUy] and b
  // (2D, box = the tile + 2-cell halo; tma_ok = 0: per-thread loads instead)
  CUtensorMap tma_state[2][3];
  CUtensorMap tma_b;
  int tma_ok = 0;
  // sources / wind
  std::vector<swf::DevSrc> h_src;
  std::vector<double> h_ht, h_hq;
  swf::DevSrc* d_src = nullptr;
  double* d_ht = nullptr;
  double* d_hq = nullptr;
  double* d_sig = nullptr;  // 2*nsrc: sigma at t_n, sigma at t_mid
  std::vector<double> h_wt, h_wv;
  double* d_wt = nullptr;
  double* d_wv = nullptr;  // 2 per sample
  // masks
  int* d_interior = nullptr;
  int* d_halo = nullptr;
  unsigned char* d_bflag = nullptr;  // bit0 lagrangian-active, bit1 flux-active
  unsigned char* d_tile_act = nullptr;  // 2 x tiles: [cur] this step, [1-cur] previous
  unsigned char* d_tile_same = nullptr;  // tile identical in both state buffers
  unsigned* d_tile_srcm = nullptr;       // per-tile source-spec masks (fused_tile_srcm)
  int* d_redo_f = nullptr;  // k_forces tiles to redo exactly (speculative division rejected)
  int* d_redo_s = nullptr;  // k_step tiles to redo exactly
  int* d_list_f = nullptr;  // k_forces work list
  int* d_list_s = nullptr;  // k_step work list
  int* d_redo_l = nullptr;  // k_lag tiles to redo exactly (split step)
  // split step (SWF_SPLIT): the half-step view (depth, u, v) k_lag leaves for
  // k_flux, local cells each
  double* d_half[3] = {nullptr, nullptr, nullptr};
  // exact StepInfo volumes (full grids): k_step stores the terms of the
  // reference's volume sums; fused_exact_volumes adds them in its order
  double* d_xdef = nullptr;    // clamp deficit per cell (flux-on cells of the step)
  double* d_xsrc = nullptr;    // Ht - Hn per cell (active cells of the step)
  double* d_xbpart = nullptr;  // 2 per owned block: deficit, source partials
  double* d_xface = nullptr;   // [W ny | E ny | S nx | N nx] boundary fm
  int sm_count = 148;
  swf::FaceTaps taps;  // owned by the nests that registered them
  // P2P halo: the neighbours' state buffers mapped here ([side][field][parity])
  double* peer[2][3][2] = {};
  int peer_on[2] = {0, 0};
  int peer_drow[2] = {0, 0};
  double* d_part = nullptr;              // per-tile diagnostic partials (3 per tile)
  // scalars
  swf::StepScalars* d_sc = nullptr;
  swf::StepScalars* h_sc = nullptr;  // pinned mirror
  double h_t = 0.0;                  // host copy of t after the last sync
  // stage path
  swf::Scratch* scr = nullptr;
  int mode = 0;  // 0 fused, 1 staged
  int batch_cur0 = -1;  // asynchronous strip batch: ping-pong index at its start
  // after a sparse-ingest host-buffer step the device holds the momentum of
  // the flux-active tiles only: resident calls need a fresh upload first
  int state_partial = 0;
  double* wt_host[3] = {nullptr, nullptr, nullptr};  // write-through targets of a host step
  // opt-in host mirror (swf_set_host_mirror): the caller's pinned arrays
  // equal the device state after the last host step (SURVEY.md 8b Ownership)
  int host_mirror = 0;
  int mirror_valid = 0;
  const double* mirror_ptr[3] = {nullptr, nullptr, nullptr};
  double mirror_t = 0.0;
  long long last_ingest_bytes = 0;
  int batch_steps = 0;
  int last_staged = 0;  // which path produced the last diagnostics
  int defer_volumes = 0;  // swf_step leaves the exact volumes to its caller (nested coupling)
  // timing
  bool timing = false;
  cudaEvent_t ev[10] = {};
  // per-step event ring of the fused path (swf_set_timing(ctx, slots))
  std::vector<cudaEvent_t> tev;  // 6 per slot
  int tslots = 0;
  long long tstep = 0;
  // CUDA graph of one fused step (captured lazily, invalidated on config change)
  cudaGraphExec_t graph = nullptr;
  double graph_dt_cap = -1.0;
  // pinned staging for host-buffer steps
  double* h_pin = nullptr;
  size_t h_pin_cells = 0;
  std::string err;
};

namespace swf {

// stage path (swf_stage.cu)
int stage_run(swf_ctx* c, int stage, double arg, double* tau_out);
int stage_step(swf_ctx* c, double dt_cap, swf_step_info* info);
int stage_download(swf_ctx* c, int which, double* out);
void stage_free(swf_ctx* c);

// fused path (swf_fused.cu)
int fused_enqueue_step(swf_ctx* c, double dt_cap);
int fused_prepare(swf_ctx* c);
int fused_reduce_ctas();
int fused_restore_host(swf_ctx* c, double* hH, double* hHUx, double* hHUy);
int fused_enqueue_phase1(swf_ctx* c, double dt_cap);
int fused_enqueue_phase2(swf_ctx* c, double dt_cap);
int fused_enqueue_phase2(swf_ctx* c, double dt_cap, double global_speed);
int fused_enqueue_phase2(swf_ctx* c, double dt_cap, double global_speed, const double* gspeed);
int fused_enqueue_phase1(swf_ctx* c, double dt_cap, int part);
int fused_local_speed(swf_ctx* c, double* dev_out);
int fused_ingest_hu(swf_ctx* c, const double* hHUx, const double* hHUy);
int fused_tile_srcm(swf_ctx* c);
int fused_exact_volumes(swf_ctx* c);  // enqueue the exact reduction of the last step

int launch_begin(swf_ctx* c, double dt_cap);  // sources/wind at t_n, reset counters
int launch_mask(swf_ctx* c);                   // K1 block mask + tile flags
int launch_tau(swf_ctx* c, double dt_cap);     // tau from speed_bits, then mid scalars
int launch_mid(swf_ctx* c, double tau);        // mid scalars for a given tau
void fill_block_counts(const swf_ctx* c, const StepScalars* sc, swf_step_info* info);
int stage_volumes(swf_ctx* c, double* v3);
void stage_clear_sources(swf_ctx* c);

// shared helpers (swf_capi.cu)
int set_err(swf_ctx* c, int code, const std::string& msg);
int cuda_check(swf_ctx* c, cudaError_t e, const char* what);
int check_device_error(swf_ctx* c);  // after a sync: maps err_key to status
size_t local_cells(const swf_ctx* c);
void invalidate_mask(swf_ctx* c);  // the state changed outside the fused path
void invalidate_graph(swf_ctx* c); // the captured step no longer matches the context
// a batch of enqueued steps: reset the device counters before, and after the
// synchronisation commit the steps done (ping-pong index, error status)
int batch_reset(swf_ctx* c);
int batch_commit(swf_ctx* c, int cur_start, int enqueued, int* done);
inline unsigned char* tile_act_at(swf_ctx* c, int parity) {
  return c->d_tile_act + (size_t)parity * ((size_t)c->geo.tiles_x * c->geo.tiles_y);
}

// per-cell source evaluation (sources.cpp:45-64, 66-75) on the device
__device__ __forceinline__ double cell_source(const DevSrc* src, const double* sig, int nsrc,
                                              int i, int jg, double& vx, double& vy) {
  double s = 0.0;
  for (int m = 0; m < nsrc; ++m) {
    const DevSrc& d = src[m];
    if (i >= d.i0 && i <= d.i1 && jg >= d.j0 && jg <= d.j1) {
      s += sig[m];
      vx = d.vx;
      vy = d.vy;
    }
  }
  return s;
}

__device__ __forceinline__ double cell_sigma_only(const DevSrc* src, const double* sig, int nsrc,
                                                  int i, int jg) {
  double s = 0.0;
  for (int m = 0; m < nsrc; ++m) {
    const DevSrc& d = src[m];
    if (i >= d.i0 && i <= d.i1 && jg >= d.j0 && jg <= d.j1) s += sig[m];
  }
  return s;
}

}  // namespace swf
