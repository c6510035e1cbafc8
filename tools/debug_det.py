import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_04547_b200 import engine as E, models, synth
from paper_2104_04547_b200.screen import DeviceLibrary, HostStager
vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
m = models.FusionModel(vcfg, gcfg, fcfg, seed=0)
dm = E.DeviceModel(vcfg, gcfg, fcfg, m.all_params())
B = 1024
pocket = synth.make_pocket(1000, seed=0)
lib = synth.make_poses(410, 10, seed=1000).slice(0, 2 * B)
dl = DeviceLibrary(lib, [pocket], torch.device("cuda"))
outs = ("scores", "lat_v", "lat_g")
for prec in ("fp32", "bf16"):
    runs = []
    for r in range(3):
        o = dm.score_poses(dl.batch(0, B), prec, 32768, outputs=outs, retry=False)
        runs.append({k: o[k].clone() for k in outs})
    torch.cuda.synchronize()
    for k in outs:
        d1 = (runs[0][k] - runs[1][k]).abs().max().item()
        d2 = (runs[0][k] - runs[2][k]).abs().max().item()
        print(prec, k, "run-to-run maxdiff", d1, d2)
    # sub-batch
    o = dm.score_poses(dl.batch(0, 64), prec, 32768, outputs=outs, retry=False)
    for k in outs:
        print(prec, k, "subbatch maxdiff", (o[k] - runs[0][k][:64]).abs().max().item())
