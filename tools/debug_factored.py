"""Print factored-vs-full differences on a small screen (GPU)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_04547_b200 import engine as E  # noqa: E402
from paper_2104_04547_b200 import models, synth  # noqa: E402

vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
dm = E.DeviceModel(vcfg, gcfg, fcfg, models.FusionModel(vcfg, gcfg, fcfg, seed=0).all_params())
pockets = [synth.make_pocket(1000, seed=41), synth.make_pocket(420, seed=42)]
lib = synth.concat([synth.make_poses(9, 5, seed=43, target=0),
                    synth.make_poses(6, 4, seed=44, target=1, ligand_atoms=(3, 100)),
                    synth.make_poses(2, 3, seed=45, target=0, ligand_atoms=(120, 128))])
pk = (np.concatenate([p.xyz for p in pockets]), np.concatenate([p.elem for p in pockets]),
      np.concatenate([p.role for p in pockets]), np.concatenate([[0], np.cumsum([len(p.xyz) for p in pockets])]))
b = E.batch_from_arrays(lib.xyz, lib.elem, lib.role, lib.atom_off, pocket=pk, pose_target=lib.target)
cache = dm.prepare_pockets(b.pocket_xyz, b.pocket_elem, b.pocket_role, b.pocket_off)
outs = ("scores", "lat_v", "lat_g")
full = dm.score_poses(b, "bf16", 1 << 17, outs, retry=False)
fact = dm.score_poses_cached(b, cache, 1 << 17, outs, rescore=False)
torch.cuda.synchronize()
print("err full", full["err"].abs().sum().item(), "fact", fact["err"].cpu().numpy().tolist())
for k in outs:
    a, f = full[k].cpu().numpy(), fact[k].cpu().numpy()
    print(k, "max abs", np.nanmax(np.abs(a - f)), "max |full|", np.nanmax(np.abs(a)))
print("scores full", full["scores"][:6].cpu().numpy())
print("scores fact", fact["scores"][:6].cpu().numpy())
dg = (fact["lat_g"] - full["lat_g"]).abs().max(dim=1).values.cpu().numpy()
nl = np.diff(lib.atom_off)
for p in range(len(dg)):
    print(p, "target", lib.target[p], "nL", nl[p], "dlat_g %.3g" % dg[p])
