"""Scheduling never changes results: serial vs overlapped branch schedules
(fs_set_overlap), and scorer calls from a thread pool (one CUDA stream per
thread, harness.py:374-376) vs sequential calls -- bitwise identical."""

import concurrent.futures as cf

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch

    from paper_2104_04547_b200 import _native as N
    from paper_2104_04547_b200 import complexes as cx
    from paper_2104_04547_b200 import engine as E
    from paper_2104_04547_b200 import models, synth
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    model = models.FusionModel(vcfg, gcfg, fcfg, seed=0, precision="bf16")
    pocket = synth.make_pocket(1000, seed=12)
    lib = synth.make_poses(12, 10, seed=13)
    cs = [cx.SyntheticComplex(f"p{p}", *synth.complex_arrays(pocket, lib, p), 0.0) for p in range(lib.n_poses)]
    return torch, N, E, model, pocket, lib, cs


@pytest.mark.parametrize("precision", ["bf16", "mixed", "fp32"])
def test_overlap_modes_bitwise_equal(setup, precision):
    torch, N, E, model, pocket, lib, cs = setup
    dm = model.device_model()
    b = E.batch_from_arrays(lib.xyz, lib.elem, lib.role, lib.atom_off,
                            pocket=(pocket.xyz, pocket.elem, pocket.role, np.array([0, 1000])),
                            pose_target=lib.target)
    outs = []
    for mode in (0, 1, 2):
        N.lib().fs_set_overlap(mode)
        o = dm.score_poses(b, precision, outputs=("scores", "lat_v", "lat_g"))
        torch.cuda.synchronize()
        outs.append({k: v.cpu().numpy() for k, v in o.items()})
    N.lib().fs_set_overlap(-1)
    for o in outs[1:]:
        for k in ("scores", "lat_v", "lat_g"):
            assert np.array_equal(o[k], outs[0][k]), (precision, k)


def test_threaded_scorer_calls_bitwise_equal(setup):
    torch, N, E, model, pocket, lib, cs = setup
    batches = [cs[i:i + 15] for i in range(0, len(cs), 15)]
    seq = [model.score_complexes(b)[0] for b in batches]
    with cf.ThreadPoolExecutor(4) as ex:
        par = list(ex.map(lambda b: model.score_complexes(b)[0], batches * 3))
    for i, s in enumerate(par):
        assert np.array_equal(s, seq[i % len(batches)])
