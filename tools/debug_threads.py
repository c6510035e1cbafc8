"""Reproduce scorer calls from a thread pool (run_campaign parallelism)."""
import os
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_04547_b200 import complexes as cx  # noqa: E402
from paper_2104_04547_b200 import harness, models, synth  # noqa: E402


def main():
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    model = models.FusionModel(vcfg, gcfg, fcfg, seed=0, precision="bf16")
    pocket = synth.make_pocket(1000, seed=0)
    lib = synth.make_poses(60, 10, seed=77)
    recs = [harness.PoseRecord(f"c{p // 10}", "t", p % 10,
                               cx.SyntheticComplex(f"p{p}", *synth.complex_arrays(pocket, lib, p), 0.0))
            for p in range(600)]
    scorer = harness.ModelScorer(model)
    if os.environ.get("DBG_MAIN_FIRST"):
        scorer(recs[:600])
        torch.cuda.synchronize()
        print("main ok", flush=True)
    for par in (1, 2, 4):
        try:
            preds, rep = harness.run_campaign(recs, scorer, n_jobs=8, parallelism=par, ranks_per_job=1, batch_size=56)
            print("par", par, "ok", len(preds), flush=True)
        except Exception:
            traceback.print_exc()
            print("par", par, "FAILED", flush=True)


if __name__ == "__main__":
    main()
