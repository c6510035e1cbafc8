"""Small invocations of every library entry point for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) on the B200:

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_04547_b200 import engine as E  # noqa: E402
from paper_2104_04547_b200 import models, synth  # noqa: E402


def main():
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    m = models.FusionModel(vcfg, gcfg, fcfg, seed=0)
    dm = E.DeviceModel(vcfg, gcfg, fcfg, m.all_params())
    pocket = synth.make_pocket(1000, seed=0)
    lib = synth.make_poses(1, 6, seed=1)
    pk = (pocket.xyz, pocket.elem, pocket.role, np.array([0, 1000]))
    b = E.batch_from_arrays(lib.xyz, lib.elem, lib.role, lib.atom_off, pocket=pk, pose_target=lib.target)
    out = {}
    for prec in ("bf16", "mixed", "fp32"):
        out[prec] = dm.score_poses(b, prec, outputs=("scores", "lat_v", "lat_g", "pred_v", "pred_g"))
    for prec in ("bf16", "mixed"):
        cache = dm.prepare_pockets(b.pocket_xyz, b.pocket_elem, b.pocket_role, b.pocket_off, precision=prec)
        out[prec + "_fact"] = dm.score_poses_cached(b, cache)
    g = E.scoring_graph_entries(b, 2.24, 5.22, 16384)
    fg = E.scoring_graph_entries(b, 2.24, 5.22, 16384, factored=True, max_pocket_atoms=1000)
    from paper_2104_04547_b200 import complexes as cx
    cs = [cx.SyntheticComplex(f"c{p}", *synth.complex_arrays(pocket, lib, p), 0.0) for p in range(3)]
    items = models.featurize(cs, vcfg, gcfg)
    m.precision = "bf16"
    preds, errs = m.predict_batch([(it.grid, it.graph) for it in items])
    s, i = E.topk_merge(out["bf16"]["scores"], torch.arange(6, device="cuda"), None, None, 4)
    E.best_pose(torch.zeros(6, dtype=torch.int64, device="cuda"), torch.arange(6, device="cuda"),
                out["bf16"]["scores"], 1)
    torch.cuda.synchronize()
    assert not errs and not out["bf16"]["err"].any() and not g["err"].any() and not fg["err"].any()
    print("sanitize ok", {k: float(v["scores"][0]) for k, v in out.items()}, preds[0])


if __name__ == "__main__":
    main()
