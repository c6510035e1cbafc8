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
lib = synth.make_poses(410, 10, seed=1000).slice(0, 4 * B)
dl = DeviceLibrary(lib, [pocket], torch.device("cuda"))
st = HostStager(lib, B, dl)
for i in range(4):
    a = dm.score_poses(dl.batch(i * B, (i + 1) * B), "bf16", 32768, retry=False)
    sa, ea = a["scores"].clone(), a["err"].clone()
    b, _ = st.stage(i)
    o = dm.score_poses(b, "bf16", 32768, retry=False)
    torch.cuda.synchronize()
    sb, eb = o["scores"], o["err"]
    diff = (sa - sb).abs()
    print(i, "err", int(ea.ne(0).sum()), int(eb.ne(0).sum()), "maxdiff", float(diff.nan_to_num(1e9).max()),
          "n_diff", int((sa != sb).sum()))
