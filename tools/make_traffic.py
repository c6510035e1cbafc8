"""Per-kernel DRAM traffic and on-chip pipe utilisation from ncu --set full
reports, written to profiles/<round>/ncu_traffic.json (bench.py reads it for
the roofline line's `traffic` and, for the SG-CNN, `onchip`).

    python tools/make_traffic.py profiles/r01/ncu_traffic.json rep1.ncu-rep [rep2.ncu-rep ...]

Every report is a tools/profile_step.py capture (2048 poses per launch);
single-CTA launches (pocket preparation) are skipped.
"""
import csv
import io
import json
import re
import subprocess
import sys

POSES = 2048
PIPES = {
    "smem_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_bank_conflict_wavefronts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "hmma_pipe_pct": "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "mufu_xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "tcgen05_bf16_pct": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "duration_ms": "gpu__time_duration.sum",
}


def kernels(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    for r in rows[2:]:
        yield {h: r[i] for i, h in enumerate(hdr)}


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def main(out, reports):
    res = {}
    for rep in reports:
        for k in kernels(rep):
            grid = k.get("launch__grid_size", "")
            if grid == "1":
                continue
            name = re.sub(r"^void |\(.*$", "", k["Kernel Name"]).replace("umma::", "").replace("fs::", "")
            rd, wr = num(k["dram__bytes_read.sum"]), num(k["dram__bytes_write.sum"])
            # ncu reports Mbyte / Kbyte columns per its units row; profile captures use Mbyte
            e = {"dram_read_bytes": rd * 1e6, "dram_write_bytes": wr * 1e6, "poses_per_launch": POSES,
                 "bytes_per_pose": (rd + wr) * 1e6 / POSES, "grid": grid, "source": rep}
            for key, metric in PIPES.items():
                v = num(k.get(metric, ""))
                if v is not None:
                    e[key] = v
            res[name] = e
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: round(v["bytes_per_pose"]) for k, v in res.items()}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
