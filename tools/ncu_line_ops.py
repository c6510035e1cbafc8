"""Executed warp instructions per (source line, SASS opcode) from an ncu report.

    python tools/ncu_line_ops.py report.ncu-rep OPCODE[,OPCODE..] [top]

Lists the source lines that execute the most instructions of the given
opcodes (e.g. IMAD,MOV), with the instruction count per line.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, ops, top=25):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, line, src = None, None, None, ""
    acc = defaultdict(float)
    text = {}
    tot = 0.0
    for r in csv.reader(io.StringIO(raw)):
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            line, src = r[0], r[1]
            continue
        sass = r[3].strip()
        if not sass or sass == "...":
            continue
        op = sass.split()[0]
        if op.startswith("@"):
            op = sass.split()[1]
        op = op.split(".")[0]
        try:
            n = float(r[7] or 0)
        except ValueError:
            continue
        tot += n
        if op in ops:
            key = (fname, line)
            acc[key] += n
            text[key] = src
    s = sum(acc.values())
    print(f"{','.join(ops)}: {s / max(tot, 1):.1%} of all executed instructions")
    for k, v in sorted(acc.items(), key=lambda x: -x[1])[:top]:
        print(f"{k[0]}:{k[1]:6s} {v / max(tot, 1):6.2%}  {text[k].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2].split(","), int(sys.argv[3]) if len(sys.argv) > 3 else 25)
