"""Per-source-line instruction / stall totals from an ncu report.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(path, top=30):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    fname, hdr, out = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0]:
            continue
        ie = hdr.index("Instructions Executed")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            out.append((fname, int(r[0]), r[1][:90], float(r[ie] or 0), float(r[st] or 0)))
        except ValueError:
            pass
    ti = sum(o[3] for o in out) or 1
    ts = sum(o[4] for o in out) or 1
    print(f"{'file:line':28s} {'instr%':>7s} {'stall%':>7s}  source")
    for f, ln, src, i, s in sorted(out, key=lambda o: -o[4])[:top]:
        print(f"{f + ':' + str(ln):28s} {i / ti:7.1%} {s / ts:7.1%}  {src.strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
