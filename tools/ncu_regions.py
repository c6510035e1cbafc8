"""Instruction / stall totals of an ncu report grouped by source-line regions
of one file (SASS in address order; inlined helpers are charged to the
region of the nearest preceding line of that file).

    python tools/ncu_regions.py report.ncu-rep file.cu name:lo-hi [name:lo-hi ...]
"""
import csv
import io
import subprocess
import sys


MIN_LINE = 0
SKIP = []          # (lo, hi) line ranges of inlined helpers: charged to their caller


def main(path, fname, specs):
    regions = []
    for sp in specs:
        name, rng = sp.split(":")
        lo, hi = map(int, rng.split("-"))
        regions.append((name, lo, hi))
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    cur_file, hdr, line = None, None, None
    sass = []
    for r in rows:
        if r and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r:
            continue
        if r[0]:
            if r[0].isdigit():
                line = int(r[0])
            continue
        ie = hdr.index("Instructions Executed")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        try:
            addr = int(r[2], 16)
        except ValueError:
            continue
        sass.append((addr, cur_file, line, float(r[ie] or 0), float(r[st] or 0),
                     {h: float(r[i] or 0) for i, h in reasons}))
    sass.sort()
    tot_i = sum(s[3] for s in sass) or 1
    tot_s = sum(s[4] for s in sass) or 1
    acc = {name: [0.0, 0.0, {}] for name, _, _ in regions}
    acc["other"] = [0.0, 0.0, {}]
    last = None
    for addr, f, ln, i, s, rs in sass:
        if f == fname and ln >= MIN_LINE and not any(lo <= ln <= hi for lo, hi in SKIP):
            last = ln
        reg = "other"
        if last is not None:
            for name, lo, hi in regions:
                if lo <= last <= hi:
                    reg = name
                    break
        acc[reg][0] += i
        acc[reg][1] += s
        for h, v in rs.items():
            acc[reg][2][h] = acc[reg][2].get(h, 0.0) + v
    for k, (i, s, rs) in acc.items():
        top = sorted(rs.items(), key=lambda x: -x[1])[:4]
        tops = "  ".join(f"{h[6:]} {v / max(s, 1):.0%}" for h, v in top if v > 0)
        print(f"{k:12s} instr {i / tot_i:6.1%}  stall {s / tot_s:6.1%}   {tops}")


if __name__ == "__main__":
    args = sys.argv[1:]
    while args[0].startswith("--"):
        opt = args.pop(0)
        if opt.startswith("--min-line="):
            MIN_LINE = int(opt.split("=")[1])
        elif opt.startswith("--skip="):
            lo, hi = opt.split("=")[1].split("-")
            SKIP.append((int(lo), int(hi)))
    main(args[0], args[1], args[2:])
