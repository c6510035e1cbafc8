"""A/B of SG-CNN kernel variants on the B200 (FS_GNN_VAR, split-2 path):
serial GNN stage time per 16,384 config-4 poses, and bf16 score error vs the
oracle on the config-1 slice (oracle scores cached in gpurun_out/)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

CACHE = os.path.join(ROOT, "profiles", "r02", "config1_oracle_scores.npy")


def main():
    mode = sys.argv[1]
    if mode == "oracle":
        s, rate = bench.cpu_oracle_pool(1024, bench.host_cores())
        np.save(CACHE, s)
        print(json.dumps({"oracle_rate": rate}))
        return
    import torch
    from paper_2104_04547_b200 import _native as N
    from paper_2104_04547_b200 import engine as E
    from paper_2104_04547_b200 import models, synth
    from paper_2104_04547_b200.screen import DeviceLibrary
    prec = os.environ.get("AB_PREC", "bf16")
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    m = models.FusionModel(vcfg, gcfg, fcfg, seed=0)
    dm = E.DeviceModel(vcfg, gcfg, fcfg, m.all_params())
    L = N.lib()
    L.fs_set_overlap(0)
    lib = bench.screen_library(0, 1640, seed=1).slice(0, 16384)
    pocket = synth.make_pocket(1000, seed=0)
    dlib = DeviceLibrary(lib, [pocket], torch.device("cuda", 0))
    evs = [torch.cuda.Event(enable_timing=True) for _ in N.STAGES]
    for e in evs:
        e.record()
    arr = (E.C.c_void_p * len(evs))(*[E.C.c_void_p(e.cuda_event) for e in evs])
    dm.score_poses(dlib.batch(0, 16384), prec, 32768, retry=False)
    torch.cuda.synchronize()
    tg = []
    for _ in range(4):
        L.fs_set_stage_events(arr, len(evs))
        dm.score_poses(dlib.batch(0, 16384), prec, 32768, retry=False)
        L.fs_set_stage_events(None, 0)
        torch.cuda.synchronize()
        tg.append(evs[6].elapsed_time(evs[7]))
    want = np.load(CACHE)
    pocket1, lib1 = bench.config1_slice()
    b = E.batch_from_arrays(lib1.xyz, lib1.elem, lib1.role, lib1.atom_off,
                            pocket=(pocket1.xyz, pocket1.elem, pocket1.role, np.array([0, 1000])),
                            pose_target=lib1.target)
    got = dm.score_poses(b, prec)["scores"].cpu().numpy()
    ref = os.path.join(ROOT, "gpurun_out", f"gnn_ab_scores_{prec}.npy")   # the first variant run in this box
    same = None
    if os.path.exists(ref):
        same = bool(np.array_equal(np.load(ref), got))
    else:
        np.save(ref, got)
    st = bench._rel_stats(got, want)
    top, wtop = bench._topk_idx(got, 100), bench._topk_idx(want, 100)
    st["top100_overlap"] = len(set(top.tolist()) & set(wtop.tolist())) / 100
    st["top10_equal"] = bool(np.array_equal(top[:10], wtop[:10]))
    print(json.dumps({"var": mode, "prec": prec, "gnn_ms_16384": min(tg), "bitwise_equal_first": same, "all": tg, **st}))


if __name__ == "__main__":
    main()
