"""Per-source-line shared-memory wavefronts / bank-conflict excess from an ncu report.

    python tools/ncu_smem_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(path, top=25):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, fname, out = None, None, []
    for r in rows:
        if r and r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0]:
            continue
        try:
            w = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
            x = float(r[hdr.index("L1 Wavefronts Shared Excessive")] or 0)
            i = float(r[hdr.index("L1 Wavefronts Shared Ideal")] or 0)
        except (ValueError, IndexError):
            continue
        if w:
            out.append((fname, int(r[0]), r[1][:80], w, x, i))
    tw = sum(o[3] for o in out) or 1
    tx = sum(o[4] for o in out) or 1
    print(f"total wavefronts {tw:.3e}, excessive {tx:.3e} ({tx / tw:.1%})")
    print(f"{'file:line':24s} {'wav%':>6s} {'exc%':>6s} {'exc/wav':>7s}  source")
    for f, ln, src, w, x, i in sorted(out, key=lambda o: -o[3])[:top]:
        print(f"{f + ':' + str(ln):24s} {w / tw:6.1%} {x / tx:6.1%} {x / w if w else 0:7.2f}  {src.strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
