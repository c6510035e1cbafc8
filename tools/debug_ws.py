import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_04547_b200 import engine as E, models, synth
from paper_2104_04547_b200.screen import DeviceLibrary
vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
m = models.FusionModel(vcfg, gcfg, fcfg, seed=0)
dm = E.DeviceModel(vcfg, gcfg, fcfg, m.all_params())
B = 1024
pocket = synth.make_pocket(1000, seed=0)
lib = synth.make_poses(410, 10, seed=1000).slice(0, B)
dl = DeviceLibrary(lib, [pocket], torch.device("cuda"))
snaps = []
for r in range(3):
    o = dm.score_poses(dl.batch(0, B), "bf16", 32768, outputs=("scores", "lat_v"), retry=False)
    torch.cuda.synchronize()
    snaps.append((dm._ws.clone(), o["lat_v"].clone()))
ws0, ws1, ws2 = snaps[0][0], snaps[1][0], snaps[2][0]
print("ws bytes", ws0.numel(), "lat_v diff 0-1", (snaps[0][1]-snaps[1][1]).abs().max().item(), "1-2", (snaps[1][1]-snaps[2][1]).abs().max().item())
for a, b, name in ((ws0, ws1, "0v1"), (ws1, ws2, "1v2")):
    d = (a != b).nonzero().flatten()
    if d.numel() == 0:
        print(name, "identical"); continue
    d = d.cpu().numpy()
    # cluster into ranges
    brk = np.flatnonzero(np.diff(d) > 4096)
    starts = np.r_[d[0], d[brk + 1]]; ends = np.r_[d[brk], d[-1]]
    print(name, "n diff bytes", len(d), "ranges", len(starts))
    for s, e in list(zip(starts, ends))[:12]:
        print("   ", s, e, e - s + 1)
