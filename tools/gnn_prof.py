"""Per-step SG-CNN timeline from a profiling build (FS_GNN_PROF):

    FS_BUILD_TAG=prof FS_EXTRA_FLAGS=-DFS_GNN_PROF python -m paper_2104_04547_b200.build_native
    FS_LIB=paper_2104_04547_b200/libfusionb200_prof.so python tools/gnn_prof.py

Scores 2,048 config-4 poses, then reads the clock64 timeline of the first 8
CTAs (poses): per message-passing step, the step span, the warps' busy
fraction (loop time / span), the items per warp and the gather share.
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_04547_b200 import _native as N  # noqa: E402
from paper_2104_04547_b200 import engine as E  # noqa: E402
from paper_2104_04547_b200 import models, synth  # noqa: E402
from paper_2104_04547_b200.screen import DeviceLibrary  # noqa: E402

WARPS = 24


def main():
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    m = models.FusionModel(vcfg, gcfg, fcfg, seed=0)
    dm = E.DeviceModel(vcfg, gcfg, fcfg, m.all_params())
    pocket = synth.make_pocket(1000, seed=0)
    lib = synth.make_poses(205, 10, seed=1).slice(0, 2048)
    dl = DeviceLibrary(lib, [pocket], torch.device("cuda"))
    dm.score_poses(dl.batch(0, 2048), "bf16", 32768, retry=False)
    torch.cuda.synchronize()
    buf = np.zeros((8, 12, WARPS, 7), dtype=np.uint64)
    L = N.lib()
    f = L.fs_debug_gnn_prof
    f.argtypes = [C.c_void_p]
    assert f(buf.ctypes.data) == 0
    b = buf.astype(np.int64)
    nw = int((b[0, 1, :, 0] > 0).sum())
    out = {"warps": nw, "poses": []}
    for p in range(8):
        t0 = b[p, 0, :nw, 0].min()
        emb = int(b[p, 0, :nw, 1].max() - t0)
        steps = []
        for s in range(1, 10):
            st, en = b[p, s, :nw, 0], b[p, s, :nw, 1]
            span = int(en.max() - st.min())
            busy = float(((en - st) / max(span, 1)).mean())
            steps.append({"span": span, "busy": round(busy, 3), "items": b[p, s, :nw, 2].tolist(),
                          "gather_frac": round(float(b[p, s, :nw, 3].sum() / max((en - st).sum(), 1)), 3),
                          "claim_frac": round(float(b[p, s, :nw, 4].sum() / max((en - st).sum(), 1)), 3),
                          "gru_frac": round(float(b[p, s, :nw, 5].sum() / max((en - st).sum(), 1)), 3),
                          "lo_tiles": int(b[p, s, :nw, 6].sum()),
                          "start_skew": int(st.max() - st.min())})
        pool_end = int(b[p, 10, :4, 0].max() - t0)
        setup0 = int(b[p, 11, :nw, 0].max() - b[p, 0, :nw, 1].max())
        setup1 = int(b[p, 11, :nw, 1].max() - b[p, 6, :nw, 1].max())
        pool = int(pool_end - (b[p, 11, :nw, 2].min() - t0))
        out["poses"].append({"embed": emb, "steps": steps, "total": pool_end, "setup0": setup0, "setup1": setup1,
                             "pool": pool})
    for p in out["poses"][:3]:
        print(json.dumps({k: p[k] for k in ("embed", "total", "setup0", "setup1", "pool")}))
        for s in p["steps"]:
            print("  ", json.dumps(s))
    tot = np.mean([p["total"] for p in out["poses"]])
    stp = np.mean([[s["span"] for s in p["steps"]] for p in out["poses"]], axis=0)
    print(json.dumps({"mean_total_cycles": tot, "mean_step_span": stp.tolist(),
                      "steps_share": float(stp.sum() / tot)}))


if __name__ == "__main__":
    main()
