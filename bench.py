#!/usr/bin/env python
"""Benchmark of the CSPH-TVD time step (BASELINE.json metric: cell-updates/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config C3|C2|C5|C1] [--no-skip]

N=1 runs configs[2] (C3: 16384^2 synthetic Volga-Akhtuba-like floodplain,
all physics) — the largest configuration BASELINE.json names that fits one
B200 — on one context; N>1 (torchrun, one rank per GPU) splits it into
B-aligned row strips with an NCCL halo exchange and an exact allreduce-max of
the CFL speed each step (multigpu.py).  One JSON line is printed by rank 0.

--impl reference times the reference's own CPU implementation (the compiled
reference in oracle/_ref, all host threads; the C restatement oracle/liborc.so
as a single-thread port when the reference was not compiled) on a bounded
crop of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GB = 1e9

# The CPU sample of C3/C5: 8 of the 64 tiles of 2048^2 cells, one from the
# middle of each eighth of the tiles sorted by their t = 0 flux-active block
# fraction (tools/cpu_sample_crops.py): C3 sample 0.361 vs 0.362 over all 64
# tiles; the diagonal crops used before held 0.283 (drier, which favoured the
# CPU).
SAMPLE_CROPS = {
    "C3": [(2048, 4096), (0, 4096), (2048, 0), (12288, 0), (6144, 14336), (10240, 10240),
           (0, 14336), (4096, 0)],
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)  # >= 100 timed
    p.add_argument("--warmup", type=int, default=20)  # and 20 warm-up steps
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="C3")
    p.add_argument("--no-skip", action="store_true", help="disable dry-block skipping")
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--fast", action="store_true",
                   help="the opt-in FAST build (libswflood_cuda_fast.so; tolerance-validated, "
                        "tests/test_gpu_fast.py) instead of the bit-exact default")
    return p.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = sorted(float(r[0]) for r in rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(pw) if pw else None}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp64_roof(kernel, active_cells, kernel_s):
    """The FP64-pipe roof beside the HBM one: the kernel's
    FP64-pipe instructions per active cell (ncu capture, profiles/) against
    the measured FP64 lane-op rate of this B200 (tools/fp64_peak.cu,
    profiles/fp64_peak_r3b.json: DADD/DMUL/DFMA throughput, CUDA events)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            k = json.load(f)["kernels"][kernel]
        with open(os.path.join(ROOT, "profiles", "fp64_peak_r3b.json")) as f:
            pk = json.load(f)
        ops = pk["ops"]
        # the mix is DADD/DMUL/DSETP-heavy with DFMA from the divisions: the
        # mean of the three measured rates
        peak = sum(ops[o]["lane_ops_per_s"] for o in ("DADD", "DMUL", "DFMA")) / 3.0
        lane_ops = 32.0 * k["fp64_inst_executed"]
        per_cell = lane_ops / k["cells"] if k.get("cells") else lane_ops / active_cells
        roof = peak / per_cell  # active cells per second
        achieved = active_cells / kernel_s
        return {"bound": "fp64", "unit": "active cell-updates/s",
                "fp64_lane_ops_per_active_cell": round(per_cell, 1),
                "peak_fp64_lane_ops_per_s": peak, "roof": round(roof, 1),
                "achieved": round(achieved, 1), "frac": round(achieved / roof, 4),
                "source": "profiles/fp64_peak_r3b.json (measured) + profiles/ncu_summary.json"}
    except Exception:
        return None


def ncu_traffic(kernel="k_step"):
    """DRAM bytes per launch of the kernel from the committed ncu --set full
    capture summary (profiles/), with its issue and FP64-pipe utilisation
    (the resources that actually bound this bit-exact fp64 path), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        k = d["kernels"][kernel]
        return {"bytes_per_launch": k["dram_bytes"], "source": d.get("source", p),
                "cells_per_launch": k.get("cells"),
                "fp64_pipe_pct": round(k["fp64_pipe_pct"], 1),
                "issue_active_pct": round(k["issue_active_pct"], 1)}
    except Exception:
        return None


# ---------------------------------------------------------------------------
# reference CPU arm (and cpu_baseline)
# ---------------------------------------------------------------------------
def cpu_reference(config, warmup=5, steps=30, threads=None, crop=2048):
    """The reference's CPU implementation on a bounded sample of the workload,
    stepped like the B200 arm: `warmup` untimed steps, then `steps` timed
    steps, from the same initial state (so both cover the same simulated
    window of the flood).  The sample is 8 crops of crop^2 cells along the
    diagonal of the full C3/C5 grid (same generator; the wet/dry mix of the
    domain is spatially correlated, so one crop is not representative); one
    "step" steps all 8 crops once.  Returns (Mcell-updates/s, cores, kind,
    sample description, per-step Mcell/s list)."""
    from oracle import pyorc
    from paper_1705_00614_b200 import scenarios as S
    kind = "reference" if pyorc.available("ref") else "port"
    if not pyorc.available("ref" if kind == "reference" else "orc"):
        try:
            pyorc.build(ref=False)
        except Exception:
            pass
    cores = threads or os.cpu_count() or 1
    if kind != "reference":
        cores = 1
    n_full = {"C3": 16384, "C5": 32768}.get(config, 0)
    if config == "C5W":  # the weak-scaling band: 8 crops along its 4096 rows
        c = min(crop, S.WEAK_ROWS // 2)
        wins = [(k * 4096 + 2048 - c // 2, S.WEAK_ROWS // 2 - c // 2, c, c) for k in range(8)]
        scs = [S.build("C5", window=w) for w in wins]
        n_full = 32768
    elif n_full and crop == 2048 and config in SAMPLE_CROPS:
        c = crop
        wins = [(i0, j0, c, c) for i0, j0 in SAMPLE_CROPS[config]]
        scs = [S.build(config, window=w) for w in wins]
    elif n_full:
        c = min(crop, n_full // 8)
        wins = [(k * (n_full // 8) + (n_full // 16) - c // 2,) * 2 + (c, c) for k in range(8)]
        scs = [S.build(config, window=w) for w in wins]
    else:
        scs = [S.build(config)]
    steppers = []
    for sc in scs:
        sc.options.workers = cores
        o = pyorc.OracleStepper(sc.terrain, sc.params, sc.control, sc.options,
                                kind="ref" if kind == "reference" else "orc")
        if sc.wind.any():
            o.set_wind(sc.wind)
        if sc.sources:
            o.set_sources(sc.sources)
        o.upload(sc.state)
        steppers.append(o)
    cells = sum(sc.cells() for sc in scs)
    for _ in range(warmup):
        for o in steppers:
            o.run(1)
    per_step, t_all = [], time.perf_counter()
    crop_s = [0.0] * len(steppers)
    act = [0.0] * len(steppers)
    for _ in range(steps):
        t0 = time.perf_counter()
        for q, o in enumerate(steppers):
            tq = time.perf_counter()
            _, info = o.run(1)
            crop_s[q] += time.perf_counter() - tq
            act[q] += info.active_fraction / steps
        per_step.append(cells / (time.perf_counter() - t0) / 1e6)
    el = time.perf_counter() - t_all
    for o in steppers:
        o.close()
    v = cells * steps / el / 1e6
    # the sample's activity (flux-active block fraction, StepInfo, mean over
    # the timed steps) and each crop's own rate
    detail = {"active_fraction": round(sum(a * sc.cells() for a, sc in zip(act, scs)) / cells, 4),
              "crops": [{"window": list(sc.window) if getattr(sc, "window", None) else None, "active_fraction": round(a, 4),
                         "mcells_s": round(sc.cells() * steps / t / 1e6, 3) if t > 0 else None}
                        for sc, a, t in zip(scs, act, crop_s)]}
    kind_of = ("band" if config == "C5W" else
               "stratified" if (crop == 2048 and config in SAMPLE_CROPS) else "diagonal")
    what = (f"8 {kind_of} {scs[0].terrain.nx}x{scs[0].terrain.ny} crops of {config}" if n_full
            else f"{config} full grid")
    cpu = "unknown CPU"
    try:
        with open("/proc/cpuinfo") as f:
            cpu = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    built = ("the reference sources compiled by oracle/Makefile: g++ -O3 -ffp-contract=off "
             "-fopenmp, no -march" if kind == "reference" else "the C restatement (gcc -O2)")
    sample = (f"{what} (same generator, {cells / 1e6:.1f} M cells, flux-active fraction "
              f"{detail['active_fraction']}), {warmup} warm-up + {steps} "
              f"timed steps from t=0 like the B200 arm, {el:.1f} s, {cores} thread(s) of "
              f"{os.cpu_count()} on {cpu}; {built}")
    return v, cores, ("reference" if kind == "reference" else "port"), sample, per_step, detail


def reference_arm(args):
    """bench.py --impl reference: the reference's CPU path with every host
    thread, W warm-up and K timed steps of the bounded sample (cpu_reference)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    v, cores, kind, sample, per_step, detail = cpu_reference(args.config, args.warmup, args.steps)
    line = {"metric": "cell-updates/sec (Mcells/s)", "value": round(v, 3), "unit": "Mcells/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True,
            "scaling": "weak" if args.config == "C5W" else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} (bounded sample on host CPU)", "grid": args.config},
            "cpu_baseline": {"value": round(v, 3), "unit": "Mcells/s", "cores": cores,
                             "kind": kind, "sample": sample, **detail},
            "e2e": {"value": round(v, 3), "unit": "Mcells/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def b200_single(args):
    import numpy as np
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper, scenarios as S

    torch.cuda.set_device(0)
    t_gen = time.perf_counter()
    sc = S.build(args.config, device="cuda")
    torch.cuda.empty_cache()  # the generator's device tensors: back to the driver for the contexts
    if args.no_skip:
        sc.options.skip_dry_blocks = False
    gen_s = time.perf_counter() - t_gen
    N = sc.cells()
    st = CsphTvdStepper(sc.terrain, sc.params, sc.control, sc.options)
    if sc.wind.any():
        st.set_wind(sc.wind)
    if sc.sources:
        st.set_sources(sc.sources)
    st.upload(sc.state)
    stream = torch.cuda.ExternalStream(st.stream_handle())

    # warm-up (CUDA-graph replay path)
    st.run(args.warmup)
    info = st.step_resident()  # one synchronised step: StepInfo with block counts
    K = args.steps
    st.set_timing(K)
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    done, last = st.run(K)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    assert done == K
    tk = st.timing_read(K)  # (K, 8) seconds per bucket
    st.set_timing(0)
    t_step_kernel = float(tk[:, 6].mean())
    t_forces_kernel = float(tk[:, 1].mean())

    # active cells (flux-active blocks at B=16)
    bs = sc.options.block_size
    n_act = min(N, last.flux_blocks * bs * bs) if sc.options.skip_dry_blocks else N
    has_nf = sc.params.n_field is not None
    per_act = 56 + (8 if has_nf else 0)
    alg_bytes = per_act * n_act + 8 * (N - n_act)
    hbm_peak, peak_src = peaks()
    achieved = alg_bytes / t_step_kernel / GB
    traffic = ncu_traffic("k_step") if args.config == "C3" else None  # the capture is of C3
    value = N * K / (ms * 1e-3) / 1e6

    # ---- end to end through the drop-in host-buffer step() ----
    E = max(1, args.e2e_steps)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
    from paper_1705_00614_b200.types import FlowState
    hs = FlowState(sc.terrain.nx, sc.terrain.ny, 0.0, pin(sc.state.H), pin(sc.state.HUx),
                   pin(sc.state.HUy))
    st.download(hs)  # continue from the current device state
    st.step(hs)  # warm-up of the host path
    torch.cuda.synchronize()
    d2h = h2d = 0
    t0 = time.perf_counter()
    for _ in range(E):
        st.step(hs)
        d2h += st.last_writeback_bytes() + 8  # the values k_step wrote back, + t
        h2d += st.last_ingest_bytes() + 8
    e2e_s = time.perf_counter() - t0
    e2e_value = N * E / e2e_s / 1e6

    # ---- the same host steps with the opt-in host mirror (swf_set_host_mirror):
    # the caller changes its pinned arrays only through step(), so the inputs
    # are already on the device; every step still writes its result into them
    st.set_host_mirror(True)
    st.step(hs)  # establishes the mirror (one full upload)
    torch.cuda.synchronize()
    md2h = mh2d = 0
    t0 = time.perf_counter()
    for _ in range(E):
        st.step(hs)
        md2h += st.last_writeback_bytes() + 8
        mh2d += st.last_ingest_bytes() + 8
    mirror_s = time.perf_counter() - t0
    st.set_host_mirror(False)
    e2e_mirror = {"value": round(N * E / mirror_s / 1e6, 3), "unit": "Mcells/s",
                  "h2d_bytes_per_step": int(mh2d // E), "d2h_bytes_per_step": int(md2h // E),
                  "how": "as e2e, with the opt-in host mirror (swf_set_host_mirror, SURVEY.md 8b "
                         "Ownership): the caller's pinned arrays change only through step(), so "
                         "no host->device copy is needed; k_step still writes every updated "
                         "cell into them, t read back; host-timed, synchronised"}

    cpu = None
    if not args.no_cpu_baseline:
        try:
            v, cores, kind, sample, _, detail = cpu_reference(args.config, args.warmup, args.steps)
            cpu = {"value": round(v, 3), "unit": "Mcells/s", "cores": cores, "kind": kind,
                   "sample": sample, **detail}
            # a 1-core run beside the all-threads one (a shorter
            # window: 1 warm-up + 2 timed steps of the same 8 crops)
            v1, _, _, sample1, _, _ = cpu_reference(args.config, 1, 2, threads=1)
            cpu["single_core"] = {"value": round(v1, 3), "unit": "Mcells/s", "cores": 1,
                                  "sample": sample1}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": "Mcells/s", "cores": None, "kind": None,
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": "cell-updates/sec (Mcells/s)", "value": round(value, 3), "unit": "Mcells/s",
        # the same rate over the cells of flux-active blocks
        "value_active": round(n_act * K / (ms * 1e-3) / 1e6, 3),
        "n_gpus": 1, "steps": K, "warmup": args.warmup, "ms_per_step": round(ms / K, 4),
        "higher_is_better": True, "scaling": "weak" if args.config == "C5W" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, scenarios.py)",
        "config": {"workload": ("C5W weak scaling, one GPU's share: " if args.config == "C5W" else "")
                   + f"{sc.name} {sc.terrain.nx}x{sc.terrain.ny} h={sc.terrain.h} m, " + (
                       "all physics (Manning field, wind, Coriolis, viscosity, 3 sources, open east edge)"
                       if args.config in ("C3", "C5") else
                       f"all physics (Manning field, wind, Coriolis, viscosity, {len(sc.sources)} "
                       "sources in the band, open east edge)" if args.config == "C5W" else
                       f"Manning n={sc.params.n_manning}, reflective edges"),
                   "cells": N, "active_fraction": round(last.active_fraction, 4),
                   "skip_dry_blocks": bool(sc.options.skip_dry_blocks),
                   "parallelism": "single GPU, fused tile kernels",
                   "l2": f"inputs larger than L2 ({8 * N / 2**30:.0f} GiB per field vs 126 MB L2)",
                   "parity": ("FAST build: normwise 1e-12 of the reference after N steps with tau "
                              "pinned, mask bit-exact (tests/test_gpu_fast.py)" if args.fast else
                              "bit-exact vs the reference CPU path (tests/test_gpu_parity.py)"),
                   "build": "fast" if args.fast else "exact",
                   "generation_s": round(gen_s, 1)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                     "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                     "traffic": traffic["bytes_per_launch"] if traffic else None,
                     "kernel": "k_step (fused K4..K8)",
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "bytes_per_active_cell": per_act, "active_cells": n_act,
                     "kernel_ms": round(t_step_kernel * 1e3, 4),
                     "forces_kernel_ms": round(t_forces_kernel * 1e3, 4),
                     "kernel_share_of_step": round(t_step_kernel / (ms * 1e-3 / K), 4),
                     "peak_source": peak_src,
                     "step_frac_of_hbm": round(alg_bytes / (ms * 1e-3 / K) / GB / hbm_peak, 4),
                     "ncu": ({"fp64_pipe_pct": traffic["fp64_pipe_pct"],
                              "issue_active_pct": traffic["issue_active_pct"],
                              "source": traffic["source"]} if traffic else None),
                     "binding": "FP64 issue and dependency latency, not HBM (DESIGN.md section 4)",
                     "fp64": (fp64_roof("k_step", n_act, t_step_kernel)
                              if args.config == "C3" else None)},
        "e2e": {"value": round(e2e_value, 3), "unit": "Mcells/s",
                "h2d_bytes_per_step": int(h2d // E), "d2h_bytes_per_step": int(d2h // E),
                "how": "CsphTvdStepper.step(FlowState) on pinned host buffers, every step: H and "
                       "t copied in full (copy engine), the block mask computed on the device, "
                       "HUx/HUy read over PCIe for the flux-active tiles only (every cell whose "
                       "momentum the step reads or writes back), one fused step whose k_step "
                       "writes every updated cell straight into the pinned host arrays (PCIe "
                       "writes overlapped with the arithmetic; restored on a numerical abort), "
                       "t read back; d2h counts the values written (device counter); "
                       "host-timed, synchronised"},
        "e2e_host_mirror": e2e_mirror,
        "gpu_launches": 10 * K,  # begin, flist, forces, forces_redo, tau, slist, step, step_redo, reduce, finish
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def b200_nested(args):
    """C4 (BASELINE.json configs[3]): coarse 4096^2 at 50 m + a 1024^2-cell
    window refined r=4 (4096^2 fine cells at 12.5 m + ghost band), coupled
    every global step (swf_coupled_step: global step, fine subcycling with
    time-interpolated ghosts, restriction).  value = (coarse cells + fine
    cells x fine substeps) / device time."""
    import torch
    from paper_1705_00614_b200 import CsphTvdStepper, scenarios as S
    from paper_1705_00614_b200.nesting import NestedGrid, coupled_step

    torch.cuda.set_device(0)
    t_gen = time.perf_counter()
    ns = S.nested_floodplain(device="cuda")
    torch.cuda.empty_cache()
    gen_s = time.perf_counter() - t_gen
    sc, fs = ns.coarse, ns.fine
    coarse = CsphTvdStepper(sc.terrain, sc.params, sc.control, sc.options)
    coarse.set_wind(sc.wind)
    if sc.sources:
        coarse.set_sources(sc.sources)
    coarse.upload(sc.state)
    nest = NestedGrid(coarse, ns.window, ns.r, fs.terrain, fs.params, fs.control, fs.options,
                      ghost=ns.ghost)
    nest.fine.set_wind(fs.wind)
    if fs.sources:
        nest.fine.set_sources(fs.sources)
    nest.upload(fs.state)
    Nc, Nf = sc.cells(), fs.cells()
    for _ in range(args.warmup):
        coupled_step(coarse, [nest])
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    K = args.steps
    subs = 0
    t0 = time.perf_counter()
    for _ in range(K):
        ci = coupled_step(coarse, [nest])  # synchronising (host reads fine t per substep)
        subs += ci.substeps_total
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    clk = clocks.stop()
    updates = Nc * K + Nf * subs
    value = updates / el / 1e6
    line = {
        "metric": "cell-updates/sec (Mcells/s)", "value": round(value, 3), "unit": "Mcells/s",
        "n_gpus": 1, "steps": K, "warmup": args.warmup, "ms_per_step": round(el / K * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, scenarios.nested_floodplain)",
        "config": {"workload": f"C4 nested: coarse {sc.terrain.nx}x{sc.terrain.ny} h={sc.terrain.h} m "
                               f"+ window {ns.window[2]}x{ns.window[3]} coarse cells at r={ns.r} "
                               f"({fs.terrain.nx}x{fs.terrain.ny} fine cells incl. ghost band), "
                               "coupled every global step, two-way",
                   "coarse_cells": Nc, "fine_cells": Nf,
                   "fine_substeps_per_step": round(subs / K, 3),
                   "timing": "host clock around synchronising coupled steps (device work + "
                             "per-substep host reads of the fine time)",
                   "generation_s": round(gen_s, 1)},
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def b200_multi(args):
    import torch.distributed as dist
    from paper_1705_00614_b200 import multigpu
    line = multigpu.bench_strips(args)
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def relaunch_under_torchrun(args) -> int:
    """`python bench.py --gpus N` without an external launcher: re-execute
    this script under torch.distributed.run, one rank per GPU (the driver's
    own launch line), and return its exit code.  With fewer visible GPUs than
    N the ranks share devices round-robin (the same code path)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: relaunching under torchrun with {args.gpus} ranks", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.fast:
        os.environ["SWF_FLAVOR"] = "fast"  # read when the package loads its library
    rank, world, local = dist_env()
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        reference_arm(args)
        return
    if args.config == "C4":
        b200_nested(args)
    elif world > 1 or args.gpus > 1:
        b200_multi(args)
    else:
        b200_single(args)


if __name__ == "__main__":
    main()
