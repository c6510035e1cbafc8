"""profiles/r02/ncu_traffic.json from `ncu --page raw --csv` exports of
tools/profile_step.py captures (2,048 poses per launch):

    python tools/make_traffic_r02.py out.json step_bf16_raw.csv[:bf16] gnn_mixed_raw.csv:mixed

Keys: gnn_<precision>, graph_csr, conv1..conv4, dense1, voxelize (bench.py
reads `gnn_<precision>` / `graph_csr` / `convN` for the roofline line's
`traffic` and `onchip`).
"""
import csv
import json
import sys

POSES = 2048
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
ONCHIP = {
    "smem_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_bank_conflict_wavefronts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "hmma_pipe_pct": "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "mufu_xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
}


def key_of(name, prec):
    if "gnn_mma_kernel" in name:
        return f"gnn_{prec}"
    if "graph_csr_kernel" in name:
        return "graph_csr"
    if "voxelize" in name:
        return "voxelize"
    if "dense_tf32" in name:
        return "dense1"
    if "conv_umma_kernel" in name:
        sig = name.split("Cfg<")[1].split(">")[0].replace(" ", "")
        return {"16,8,32,5": "conv1", "16,32,32,3": "conv2", "8,32,64,3": "conv3", "8,64,64,3": "conv4"}.get(
            ",".join(sig.split(",")[:4]))
    return None


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def main(out, specs):
    res = {}
    for spec in specs:
        path, _, prec = spec.partition(":")
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        col = {h: i for i, h in enumerate(hdr)}
        for r in rows[2:]:
            k = key_of(r[col["Kernel Name"]], prec or "bf16")
            if not k or k in res:
                continue
            rd = num(r[col["dram__bytes_read.sum"]]) * UNIT[units[col["dram__bytes_read.sum"]]]
            wr = num(r[col["dram__bytes_write.sum"]]) * UNIT[units[col["dram__bytes_write.sum"]]]
            e = {"kernel": r[col["Kernel Name"]][:120], "poses_per_launch": POSES, "dram_read_bytes": rd,
                 "dram_write_bytes": wr, "bytes_per_pose": (rd + wr) / POSES,
                 "duration_ms": num(r[col["gpu__time_duration.sum"]]), "source": path}
            e["onchip"] = {n: round(num(r[col[m]]), 2) for n, m in ONCHIP.items() if m in col and num(r[col[m]]) is not None}
            res[k] = e
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: round(v["bytes_per_pose"]) for k, v in res.items()}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
