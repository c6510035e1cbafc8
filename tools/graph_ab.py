"""Serial featurize-stage time (voxelizer + fused radius graph) per 16,384
config-4 poses for an FS_LIB build, and a bitwise check of the scores
against the default build's (the scoring-path CSR order is part of the
result).  AB_CACHED=1: the pocket-factored path (fs_score_poses_cached),
whole-call time."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import torch
    from paper_2104_04547_b200 import _native as N
    from paper_2104_04547_b200 import engine as E
    from paper_2104_04547_b200 import models, synth
    from paper_2104_04547_b200.screen import DeviceLibrary
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    m = models.FusionModel(vcfg, gcfg, fcfg, seed=0)
    dm = E.DeviceModel(vcfg, gcfg, fcfg, m.all_params())
    L = N.lib()
    L.fs_set_overlap(0)
    lib = bench.screen_library(0, 1640, seed=1).slice(0, 16384)
    pocket = synth.make_pocket(1000, seed=0)
    dlib = DeviceLibrary(lib, [pocket], torch.device("cuda", 0))
    if os.environ.get("AB_CACHED") == "1":
        cache = dm.prepare_pockets(dlib.pocket_xyz, dlib.pocket_elem, dlib.pocket_role, dlib.pocket_off)
        call = lambda: dm.score_poses_cached(dlib.batch(0, 16384), cache, 32768, rescore=False)  # noqa: E731
        out = call()
        t = []
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            out = call()
            e1.record()
            torch.cuda.synchronize()
            t.append(e0.elapsed_time(e1))
        s = out["scores"].float().cpu().numpy()
        ref = os.path.join(ROOT, "gpurun_out", "graph_ab_cached_scores.npy")
        same = bool(np.array_equal(np.load(ref), s)) if os.path.exists(ref) else np.save(ref, s)
        print(json.dumps({"var": sys.argv[1], "cached_ms_16384": min(t), "all": t, "scores_bitwise_equal_first": same}))
        return
    evs = [torch.cuda.Event(enable_timing=True) for _ in N.STAGES]
    for e in evs:
        e.record()
    arr = (E.C.c_void_p * len(evs))(*[E.C.c_void_p(e.cuda_event) for e in evs])
    out = dm.score_poses(dlib.batch(0, 16384), "bf16", 32768, retry=False)
    torch.cuda.synchronize()
    t = []
    for _ in range(4):
        L.fs_set_stage_events(arr, len(evs))
        out = dm.score_poses(dlib.batch(0, 16384), "bf16", 32768, retry=False)
        L.fs_set_stage_events(None, 0)
        torch.cuda.synchronize()
        t.append(evs[0].elapsed_time(evs[1]))
    s = out["scores"].float().cpu().numpy()
    ref = os.path.join(ROOT, "gpurun_out", "graph_ab_scores.npy")
    same = None
    if os.path.exists(ref):
        same = bool(np.array_equal(np.load(ref), s))
    else:
        np.save(ref, s)
    print(json.dumps({"var": sys.argv[1], "featurize_ms_16384": min(t), "all": t, "scores_bitwise_equal_first": same}))


if __name__ == "__main__":
    main()
