"""Attribute an ncu SASS source page (per-instruction executed counts and stall
samples) to the kernel's own source lines, through nvdisasm's inline line
info (developer tool).

    ncu -i prof.ncu-rep --page source --csv --kernel-name regex:k_step \
        --print-source sass > /tmp/k_step.csv
    python tools/sass_lines.py /tmp/k_step.csv k_step [ranges]

ranges: comma-separated name=first-last line ranges of swf_fused.cu to sum
(e.g. "1a=637-667,1b=668-712"); without it the top lines are printed.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.environ.get("SWF_LIB") or os.path.join(ROOT, "paper_1705_00614_b200", "libswflood_cuda.so")


def _wrapper_lines(src):
    """Lines of kernel wrappers that only call a *_tile<SPEC> body: attribution
    skips them and uses the next frame inward."""
    path = os.path.join(ROOT, "paper_1705_00614_b200", "csrc", src)
    try:
        lines = open(path).read().splitlines()
    except OSError:
        return set()
    return {i for i, l in enumerate(lines, 1) if "_tile<" in l}


def sass_lines(kernel, cubin_name="swf_fused.sm_100a.cubin", src="swf_fused.cu"):
    """offset -> (outermost non-wrapper line in src, opcode) for the kernel."""
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=d, check=True, capture_output=True)
    txt = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cubin_name)],
                         capture_output=True, text=True).stdout
    skip = _wrapper_lines(src)
    out, cur, on, chain, fresh = {}, None, False, [], True
    for ln in txt.splitlines():
        if ln.startswith(".text.") or ln.startswith("_Z"):
            on = (kernel in ln) and ln.rstrip().endswith(":") and not ln.startswith(".text.")
            continue
        if not on:
            continue
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)(.*)', ln)
        if m:
            if fresh:
                chain, fresh = [], False
            if m.group(1) == src:
                chain.append(int(m.group(2)))  # innermost first, outermost last
            frames = [l for l in chain if l not in skip]
            if frames:
                cur = frames[-1]
            continue
        fresh = True
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins = re.sub(r"^@!?U?P\w+\s+", "", m.group(2).strip())
            out[int(m.group(1), 16)] = (cur, ins.split(" ")[0].split(".")[0])
    return out


def main():
    path, kernel = sys.argv[1], sys.argv[2]
    ranges = []
    if len(sys.argv) > 3:
        for part in sys.argv[3].split(","):
            name, span = part.split("=")
            a, b = span.split("-")
            ranges.append((name, int(a), int(b)))
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    body = [r for r in rows[2:] if len(r) == len(hdr) and r[ix["Instructions Executed"]].isdigit()]
    base = int(body[0][ix["Address"]], 16)
    amap = sass_lines(kernel)
    per_line = collections.Counter()
    per_line_s = collections.Counter()
    per_line_fp = collections.Counter()
    tot = ts = 0
    for r in body:
        off = int(r[ix["Address"]], 16) - base
        line, op = amap.get(off, (None, "?"))
        n = int(r[ix["Instructions Executed"]])
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        per_line[line] += n
        per_line_s[line] += s
        if op in ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX"):
            per_line_fp[line] += n
        tot += n
        ts += s
    print(f"{kernel}: {tot} warp instructions, {ts} stall samples")
    if ranges:
        for name, a, b in ranges:
            n = sum(v for k, v in per_line.items() if k is not None and a <= k <= b)
            s = sum(v for k, v in per_line_s.items() if k is not None and a <= k <= b)
            f = sum(v for k, v in per_line_fp.items() if k is not None and a <= k <= b)
            print(f"  {name:12s} inst {n / tot * 100:5.1f}%  fp64 {f / max(n, 1) * 100:5.1f}% "
                  f"of it  stalls {s / ts * 100:5.1f}%")
    else:
        for line, n in per_line.most_common(40):
            print(f"  line {line}: inst {n / tot * 100:5.1f}%  fp64 {per_line_fp[line] / max(n, 1) * 100:5.1f}%"
                  f"  stalls {per_line_s[line] / ts * 100:5.1f}%")


if __name__ == "__main__":
    main()
