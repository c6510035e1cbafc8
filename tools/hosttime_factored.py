import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2104_04547_b200 import engine as E, models, synth
from paper_2104_04547_b200.screen import DeviceLibrary
B=16384; K=8
vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
dm = E.DeviceModel(vcfg, gcfg, fcfg, models.FusionModel(vcfg, gcfg, fcfg, seed=0).all_params())
pocket = synth.make_pocket(1000, seed=0)
lib = synth.make_poses(K*B//10+1, 10, seed=1000, ligand_atoms=(16, 64)).slice(0, K*B)
dl = DeviceLibrary(lib, [pocket], torch.device("cuda"))
cache = dm.prepare_pockets(dl.pocket_xyz, dl.pocket_elem, dl.pocket_role, dl.pocket_off)
for rep in range(3):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K+1)]
    ht = []
    ev[0].record()
    for i in range(K):
        t0 = time.perf_counter()
        out = dm.score_poses_cached(dl.batch(i*B, (i+1)*B), cache, 32768, rescore=False)
        ht.append((time.perf_counter()-t0)*1e3)
        ev[i+1].record()
    torch.cuda.synchronize()
    print("host ms", [round(x,2) for x in ht], "gpu ms", [round(ev[i].elapsed_time(ev[i+1]),2) for i in range(K)], flush=True)
