"""torchrun worker for tests/test_gpu_multirank.py (one process per GPU, NCCL).

Each rank scores its compound-aligned shard of one library with the device
Screen (pose top-k + per-compound best pose), the per-rank top-k lists are
merged over NCCL (screen.merge_topk_across_ranks), and rank 0 checks the
merged pose and compound top-k against a single-device sort of every pose's
score: bitwise equal indices and scores.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2104_04547_b200 import engine as E
    from paper_2104_04547_b200 import harness, models, synth
    from paper_2104_04547_b200.screen import DeviceLibrary, Screen, merge_topk_across_ranks
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n_comp = int(os.environ.get("FS_TEST_COMPOUNDS", "301"))
    k = 50
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    dm = E.DeviceModel(vcfg, gcfg, fcfg, models.FusionModel(vcfg, gcfg, fcfg, seed=0).all_params(), device=dev)
    pocket = synth.make_pocket(1000, seed=3)
    lib = synth.make_poses(n_comp, 10, seed=4)
    s, e = harness.compound_aligned_bounds(lib.compound, world)[rank]
    res = {"rank": rank, "shard": [s, e]}
    if e > s:
        part = lib.slice(s, e)
        dlib = DeviceLibrary(part, [pocket], dev, index_base=s)
        c0, c1 = int(part.compound[0]), int(part.compound[-1]) + 1
        out = Screen(dm, "bf16", batch_size=997, k=k).run(dlib, best_compounds=c1 - c0, compound_base=c0)
        ts, ti = out["topk_scores"], out["topk_idx"]
        cs, ci = out["topk_compound_scores"], out["topk_compound_idx"]
    else:
        ts = ti = cs = ci = None
    gs, gi = merge_topk_across_ranks(ts, ti, k, device=dev)
    gcs, gci = merge_topk_across_ranks(cs, ci, k, device=dev)
    torch.cuda.synchronize()
    if rank == 0:
        # single device: every pose's score, sorted by (score desc, index asc)
        dlib = DeviceLibrary(lib, [pocket], dev)
        allv = Screen(dm, "bf16", batch_size=1500, k=k).run(dlib, keep_scores=True, best_compounds=n_comp)
        sc = allv["scores"].cpu().numpy()
        order = np.lexsort((np.arange(len(sc)), -sc.astype(np.float64)))[:k]
        gi_, gs_ = gi.cpu().numpy(), gs.cpu().numpy()
        m = len(order)      # fewer than k poses in total: the merge pads with (NaN, int64 max)
        res["pose_topk_equal"] = bool(np.array_equal(gi_[:m], order)) and bool(np.array_equal(gs_[:m], sc[order])) \
            and bool(np.isnan(gs_[m:]).all()) and bool((gi_[m:] == np.iinfo(np.int64).max).all())
        wci, wcs = allv["topk_compound_idx"].cpu().numpy(), allv["topk_compound_scores"].cpu().numpy()
        gci_, gcs_ = gci.cpu().numpy(), gcs.cpu().numpy()
        mc = len(wci)
        res["compound_topk_equal"] = bool(np.array_equal(gci_[:mc], wci)) and bool(np.array_equal(gcs_[:mc], wcs)) \
            and bool(np.isnan(gcs_[mc:]).all())
        res["top3"] = gi[:3].tolist()
    out = os.environ.get("FS_TEST_OUT")
    if out:
        with open(os.path.join(out, f"rank{rank}.json"), "w") as fh:
            json.dump(res, fh)
    print("RESULT " + json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
