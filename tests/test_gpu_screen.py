"""GPU: the screening loop.

- streaming a packed library through pinned staging gives bitwise the same
  scores and top-k as the HBM-resident library;
- the per-compound best pose folded on device batch by batch equals the
  reference rule (evaluate.aggregate_best_pose, evaluate.py:67-83, restated
  in oracle.best_pose) applied to the same scores, including ties;
- the top-k over compounds equals the oracle top-k of those best scores."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import fusion_oracle as orc  # noqa: E402


@pytest.fixture(scope="module")
def setup():
    import torch  # noqa: F401

    from paper_2104_04547_b200 import engine as E
    from paper_2104_04547_b200 import models, screen, synth
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    dm = E.DeviceModel(vcfg, gcfg, fcfg, models.FusionModel(vcfg, gcfg, fcfg, seed=0).all_params())
    pockets = [synth.make_pocket(700, seed=31, name="a"), synth.make_pocket(350, seed=32, name="b")]
    lib = synth.concat([synth.make_poses(23, 7, seed=33, target=0),
                        synth.make_poses(17, 5, seed=34, target=1, compound_base=23)])
    return E, screen, dm, pockets, lib


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_streamed_equals_resident_and_best_pose(setup, tmp_path, precision):
    import torch

    from paper_2104_04547_b200 import poselib
    E, screen, dm, pockets, lib = setup
    if not dm.supports(precision):
        pytest.skip(f"{precision} unsupported")
    sc = screen.Screen(dm, precision=precision, batch_size=37, k=20)
    dlib = screen.DeviceLibrary(lib, pockets, torch.device("cuda"), index_base=1000)
    a = sc.run(dlib, keep_scores=True, best_compounds=40)

    path = tmp_path / "lib.fspl"
    poselib.save_library(path, pockets, lib)
    pk2, lib2 = poselib.load_library(path)
    loader = poselib.StreamingLoader(lib2, pk2, 37, index_base=1000)
    b = sc.run(loader, keep_scores=True, best_compounds=40)
    torch.cuda.synchronize()
    assert loader.h2d_bytes > 0
    for k in ("scores", "topk_scores", "topk_idx", "best_score", "best_pose", "topk_compound_idx"):
        assert torch.equal(a[k].cpu(), b[k].cpu()) or (
            k.endswith("score") and torch.equal(a[k].cpu().nan_to_num(7), b[k].cpu().nan_to_num(7))), k
    assert int(a["err"].abs().sum()) == 0

    s = a["scores"].cpu().numpy()
    want = orc.best_pose(lib.compound.tolist(), [0] * lib.n_poses, lib.pose_id.tolist(), s.tolist())
    bs, bp = a["best_score"].cpu().numpy(), a["best_pose"].cpu().numpy()
    for c in range(40):
        assert (int(bp[c]), float(bs[c])) == want[(c, 0)], c
    ws, wi = orc.topk(bs, 20)
    assert np.array_equal(a["topk_compound_idx"].cpu().numpy(), wi)
    assert np.array_equal(a["topk_compound_scores"].cpu().numpy(), ws.astype(np.float32))
    ps, pi = orc.topk(s, 20, index_base=1000)
    assert np.array_equal(a["topk_idx"].cpu().numpy(), pi)


def test_best_pose_accumulator_streams_ties_and_ranges(setup):
    import torch
    E = setup[0]
    rng = np.random.default_rng(7)
    n = 5000
    comp = rng.integers(90, 160, size=n)             # some outside [100, 150)
    pid = rng.integers(0, 12, size=n)
    sc = rng.integers(-5, 5, size=n).astype(np.float32)
    sc[::97] = np.nan
    for direction in ("max", "min"):
        acc = E.BestPoseAccumulator(50, compound_base=100, direction=direction)
        for s in range(0, n, 613):                     # ragged batches
            e = min(n, s + 613)
            acc.update(torch.from_numpy(comp[s:e]).cuda(), torch.from_numpy(pid[s:e]).cuda(),
                       torch.from_numpy(sc[s:e]).cuda())
        bs, bp = (t.cpu().numpy() for t in acc.result())
        keep = (comp >= 100) & (comp < 150) & ~np.isnan(sc)
        want = orc.best_pose(comp[keep].tolist(), [0] * int(keep.sum()), pid[keep].tolist(), sc[keep].tolist(),
                             direction)
        for c in range(50):
            if (c + 100, 0) in want:
                assert (int(bp[c]), float(bs[c])) == want[(c + 100, 0)], (direction, c)
            else:
                assert bp[c] == -1 or np.isnan(bs[c])


def test_empty_compound_reports_no_pose(setup):
    import torch
    E = setup[0]
    acc = E.BestPoseAccumulator(3)
    acc.update(torch.tensor([0, 2], device="cuda"), torch.tensor([4, 5], device="cuda"),
               torch.tensor([1.5, -2.0], device="cuda"))
    bs, bp = (t.cpu().numpy() for t in acc.result())
    assert bp.tolist() == [4, -1, 5]
    assert bs[0] == np.float32(1.5) and np.isnan(bs[1]) and bs[2] == np.float32(-2.0)


def test_factored_screen_matches_full_screen(setup):
    import torch
    E, screen, dm, pockets, lib = setup
    if not dm.supports("bf16"):
        pytest.skip("bf16 unsupported")
    dlib = screen.DeviceLibrary(lib, pockets, torch.device("cuda"))
    cache = dm.prepare_pockets(dlib.pocket_xyz, dlib.pocket_elem, dlib.pocket_role, dlib.pocket_off)
    full = screen.Screen(dm, "bf16", batch_size=50, k=15).run(dlib, keep_scores=True, best_compounds=40)
    fact = screen.Screen(dm, "bf16", batch_size=50, k=15, pocket_cache=cache).run(dlib, keep_scores=True,
                                                                                 best_compounds=40)
    assert int(fact["err"].abs().sum()) == 0
    assert (fact["scores"] - full["scores"]).abs().max().item() < 2e-6
    assert torch.equal(fact["topk_idx"], full["topk_idx"])
    assert torch.equal(fact["best_pose"], full["best_pose"])
    assert torch.equal(fact["topk_compound_idx"], full["topk_compound_idx"])


def test_concurrent_scoring_threads_bitwise():
    """The reference calls scorer plugins concurrently from a thread pool
    (harness.py:374-376; frozen models are safe for concurrent
    read-only prediction).  Four host threads, each on its own CUDA stream,
    score different batches with one DeviceModel: every result equals the
    sequential one bitwise (per-thread workspaces, read-only weight blob)."""
    import threading

    import torch

    from paper_2104_04547_b200 import engine as E
    from paper_2104_04547_b200 import models, synth
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    dm = E.DeviceModel(vcfg, gcfg, fcfg, models.FusionModel(vcfg, gcfg, fcfg, seed=0).all_params())
    pocket = synth.make_pocket(1000, seed=31)
    pk = (pocket.xyz, pocket.elem, pocket.role, np.array([0, 1000]))
    batches = []
    for k in range(4):
        lib = synth.make_poses(6 + k, poses_per_compound=5, seed=40 + k)
        batches.append(E.batch_from_arrays(lib.xyz, lib.elem, lib.role, lib.atom_off, pocket=pk,
                                           pose_target=lib.target))
    want = [dm.score_poses(b, "bf16")["scores"].cpu().numpy() for b in batches]
    got = [None] * 4
    errors = []

    def work(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    out = dm.score_poses(batches[k], "bf16")["scores"]
                s.synchronize()
                got[k] = out.cpu().numpy()
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k in range(4):
        assert np.array_equal(got[k], want[k]), k
