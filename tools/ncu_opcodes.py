"""Executed warp instructions per SASS opcode (and stall samples) of one
kernel in an ncu report (captured with --import-source on / -lineinfo).

    python tools/ncu_opcodes.py report.ncu-rep [top] [--per N]

--per N divides the instruction counts by N (e.g. the poses of the launch).
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, top=40, per=1.0):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = None
    ins = defaultdict(float)
    st = defaultdict(float)
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        src = r[1].strip()
        if not src:
            continue
        op = src.split()[0]
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        ins[op] += float(r[hdr.index("Instructions Executed")] or 0)
        st[op] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    ti = sum(ins.values()) or 1
    ts = sum(st.values()) or 1
    print(f"total warp instructions {ti / per:,.0f}" + (f" per unit (/{per:g})" if per != 1 else ""))
    print(f"{'opcode':12s} {'instr':>12s} {'instr%':>7s} {'stall%':>7s}")
    for op, v in sorted(ins.items(), key=lambda x: -x[1])[:top]:
        print(f"{op:12s} {v / per:12,.0f} {v / ti:7.1%} {st[op] / ts:7.1%}")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    per = 1.0
    if "--per" in sys.argv:
        per = float(sys.argv[sys.argv.index("--per") + 1])
        args = [a for a in args if a != sys.argv[sys.argv.index("--per") + 1]]
    main(args[0], int(args[1]) if len(args) > 1 else 40, per)
