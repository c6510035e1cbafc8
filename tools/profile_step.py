"""One bf16 scoring step on a synthetic pocket screen (for ncu captures)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_04547_b200 import engine as E  # noqa: E402
from paper_2104_04547_b200 import models, synth  # noqa: E402
from paper_2104_04547_b200.screen import DeviceLibrary  # noqa: E402

B = int(os.environ.get("FS_PROFILE_BATCH", "2048"))
prec = os.environ.get("FS_PROFILE_PRECISION", "bf16")
vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
m = models.FusionModel(vcfg, gcfg, fcfg, seed=0)
dm = E.DeviceModel(vcfg, gcfg, fcfg, m.all_params())
pocket = synth.make_pocket(1000, seed=0)
lib = synth.make_poses((2 * B) // 10 + 1, 10, seed=1).slice(0, 2 * B)
dl = DeviceLibrary(lib, [pocket], torch.device("cuda"))
fact = os.environ.get("FS_PROFILE_FACTORED") == "1"
cache = dm.prepare_pockets(dl.pocket_xyz, dl.pocket_elem, dl.pocket_role, dl.pocket_off) if fact else None
for i in range(2):
    if fact:
        out = dm.score_poses_cached(dl.batch(i * B, (i + 1) * B), cache, 32768, rescore=False)
    else:
        out = dm.score_poses(dl.batch(i * B, (i + 1) * B), prec, 32768, retry=False)
torch.cuda.synchronize()
assert int(out["err"].abs().sum()) == 0
print("ok", float(out["scores"].float().mean()))
