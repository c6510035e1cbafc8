"""Stress the multi-threaded plugin path (run_campaign thread pool, one CUDA
stream per scorer thread) after large single-thread calls, as bench.py's
plugin leg does; prints the failing CUDA call site if any."""
import os
import sys
import traceback

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_04547_b200 import complexes as cx  # noqa: E402
from paper_2104_04547_b200 import harness, models, synth  # noqa: E402


def main():
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    model = models.FusionModel(vcfg, gcfg, fcfg, seed=0, precision="bf16")
    pocket = synth.make_pocket(1000, seed=0)
    lib = synth.make_poses(420, 10, seed=77)
    recs = [harness.PoseRecord(f"c{p // 10}", "t", p % 10,
                               cx.SyntheticComplex(f"p{p}", *synth.complex_arrays(pocket, lib, p), 0.0))
            for p in range(4200)]
    scorer = harness.ModelScorer(model)
    fails = 0
    for it in range(int(os.environ.get("STRESS_ITERS", "12"))):
        try:
            scorer(recs[:4096])
            torch.cuda.synchronize()
            for par in (1, 4, 8):
                preds, rep = harness.run_campaign(recs, scorer, n_jobs=16, parallelism=par, ranks_per_job=1,
                                                  batch_size=56)
                assert len(preds) == len(recs)
        except Exception:
            fails += 1
            traceback.print_exc()
    print("stress iterations done, failures:", fails, flush=True)


if __name__ == "__main__":
    main()
