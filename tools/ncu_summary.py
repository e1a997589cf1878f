"""Distil an ncu --set full report and a launch list into profiles/ (developer tool).

    python tools/ncu_summary.py gpurun_out/r1b TAG

Writes profiles/ncu_details_TAG.csv (the raw page of the captured kernels,
key metrics only), profiles/launch_shares_TAG.json (per-kernel share of the
launch list) and updates profiles/ncu_summary.json (read by bench.py for
roofline.traffic)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
         "msecond": 1.0, "second": 1e3}


def short(name):
    """Base kernel name; the persistent work-list launches report as the
    kernel they run (k_step_list -> k_step, k_forces_list -> k_forces)."""
    n = name.split("(")[0].split("::")[-1]
    return n[:-5] if n in ("k_step_list", "k_forces_list") else n


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    ix = {h: j for j, h in enumerate(hdr)}
    t, n = collections.Counter(), collections.Counter()
    for r in rows[i + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1e-6)
        t[short(r[ix["Kernel Name"]])] += v
        n[short(r[ix["Kernel Name"]])] += 1
    step = {k: v for k, v in t.items() if k.startswith("k_") and k != "k_scatter_host"}
    tot = sum(step.values())
    return {"step_kernels": {k: {"launches": n[k], "ms_total": round(v, 4),
                                 "share_of_step": round(v / tot, 4)}
                             for k, v in sorted(step.items(), key=lambda x: -x[1])},
            "all_kernels_ms": {k: round(v, 4) for k, v in t.most_common()}}


FP64_OPS = ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX")


def fp64_share(rep):
    """Share of the FP64-pipe instructions (DADD, DMUL, DFMA, DSETP, DMNMX)
    among the executed warp instructions of each kernel, from the source page
    (per-SASS-instruction executed counts)."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    out, kern, hdr = {}, None, None
    tot, fp = collections.Counter(), collections.Counter()
    for r in csv.reader(io.StringIO(txt)):
        if len(r) >= 2 and r[0] == "Kernel Name":
            kern = short(r[1])
            continue
        if r and r[0] == "Address":
            hdr = {h: j for j, h in enumerate(r)}
            continue
        if kern is None or hdr is None or len(r) < len(hdr):
            continue
        n = r[hdr["Instructions Executed"]]
        if not n.isdigit():
            continue
        op = r[hdr["Source"]].strip()
        if op.startswith("@"):
            op = op.split(None, 1)[1] if " " in op else op
        op = op.split(" ")[0].split(".")[0]
        tot[kern] += int(n)
        if op in FP64_OPS:
            fp[kern] += int(n)
    for k in tot:
        out[k] = fp[k] / tot[k] if tot[k] else 0.0
    return out


def main():
    d, tag = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", os.path.join(d, "prof.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ix = {h: j for j, h in enumerate(hdr)}
    out_csv = os.path.join(ROOT, "profiles", f"ncu_details_{tag}.csv")
    with open(out_csv, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["Kernel Name"] + [k for k in KEYS if k in ix])
        w.writerow(["unit"] + [units[ix[k]] for k in KEYS if k in ix])
        for r in rows[2:]:
            w.writerow([short(r[ix["Kernel Name"]])] + [r[ix[k]] for k in KEYS if k in ix])
    summ = {"source": f"profiles/ncu_details_{tag}.csv (ncu --set full --clock-control none, "
                      f"C3 16384^2, build {tag})", "kernels": {}}
    share = fp64_share(os.path.join(d, "prof.ncu-rep"))
    for r in rows[2:]:
        k = short(r[ix["Kernel Name"]])

        def g(m):
            return float(r[ix[m]].replace(",", "")) * (SCALE.get(units[ix[m]], 1)
                                                        if "bytes" in m else 1)
        summ["kernels"][k] = {
            "duration_ms": g("gpu__time_duration.sum") * SCALE.get(units[ix["gpu__time_duration.sum"]], 1),
            "dram_bytes": g("dram__bytes_read.sum") + g("dram__bytes_write.sum"),
            "registers": g("launch__registers_per_thread"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "inst_executed": g("smsp__inst_executed.sum"),
            # FP64-pipe warp instructions per launch (source-page share x total)
            "fp64_inst_executed": round(g("smsp__inst_executed.sum") * share.get(k, 0.0)),
        }
    lp = os.path.join(d, "launches.csv")
    if os.path.exists(lp):
        sh = launch_shares(lp)
        with open(os.path.join(ROOT, "profiles", f"launch_shares_{tag}.json"), "w") as f:
            json.dump(sh, f, indent=1)
        summ["launch_shares"] = sh["step_kernels"]
    with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
