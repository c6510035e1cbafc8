"""The drop-in boundary takes the reference's own objects (CPU only).

The reference's featurizer output (fusionscreen.models.featurize ->
VoxelGrid / ComplexGraph), its SyntheticComplex and its checkpoints must go
through this package's predict_batch / ModelScorer / load unchanged
(/root/reference/pkg/src/fusionscreen/models.py:470-529, harness.py:224-234,
checkpoint.py:48-71).  Tests that import the reference skip on the GPU box,
where it does not exist; the GPU twin (a foreign class with the same
attributes) is tests/test_gpu_parity.py::test_foreign_payload_classes."""

import os
import sys

import numpy as np
import pytest

from paper_2104_04547_b200 import complexes as cx
from paper_2104_04547_b200 import harness, models
from paper_2104_04547_b200.models import GraphHeadConfig, VoxelHeadConfig, table_coherent_fusion_config


def _ref():
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not present (GPU box)")
    if src not in sys.path:
        sys.path.append(src)
    import fusionscreen.checkpoint as ck
    import fusionscreen.complexes as rc
    import fusionscreen.models as rm
    return rc, rm, ck


def _model():
    return models.FusionModel(VoxelHeadConfig(), GraphHeadConfig(), table_coherent_fusion_config(), seed=0)


def test_reference_featurized_items_validate():
    rc, rm, _ = _ref()
    cs = [rc.generate_complex(s) for s in range(3)]
    items = rm.featurize(cs, rm.VoxelHeadConfig(), rm.GraphHeadConfig())
    m = _model()
    for it in items:
        assert m._validate_item((it.grid, it.graph)) is None


def test_validation_order_and_reasons_match_reference():
    """Items with several faults get the reference's first reason
    (models.py:515-528: shape, grid finite, feature width, features finite)."""
    rc, rm, _ = _ref()
    ref = rm.FusionModel(rm.VoxelHeadConfig(), rm.GraphHeadConfig(), rm.table_coherent_fusion_config(), seed=0)
    m = _model()
    good = rm.featurize([rc.generate_complex(1)], rm.VoxelHeadConfig(), rm.GraphHeadConfig())[0]
    grid_nan = good.grid.occupancy.copy()
    grid_nan[0, 0, 0, 0] = np.nan
    feats_bad = np.zeros((3, 5))
    feats_inf = good.graph.node_features.copy()
    feats_inf[0, 0] = np.inf
    g = good.graph

    def graph(f):
        return rc.ComplexGraph(f, g.covalent_edges, g.noncovalent_edges, g.covalent_dists, g.noncovalent_dists)
    cases = [(rc.VoxelGrid(grid_nan), graph(feats_bad)),          # both faults: grid first
             (rc.VoxelGrid(grid_nan), g),
             (good.grid, graph(feats_bad)),
             (good.grid, graph(feats_inf)),
             (rc.VoxelGrid(np.zeros((2, 4, 4, 4))), graph(feats_bad)),
             ("not a pair",), 7]
    for item in cases:
        assert m._validate_item(item) == ref._validate_item(item), item


def test_model_scorer_routes_reference_payloads():
    rc, rm, _ = _ref()
    calls = []

    class Fake:
        def score_complexes(self, cs):
            calls.append(("raw", len(cs)))
            return np.arange(len(cs), dtype=np.float64), np.zeros(len(cs), dtype=np.int32)

        def predict_batch(self, items):
            calls.append(("pairs", len(items)))
            return [1.0] * len(items), []

    sc = harness.ModelScorer(Fake())
    raw = [harness.PoseRecord("c", "t", i, rc.generate_complex(i)) for i in range(3)]
    assert sc(raw) == [0.0, 1.0, 2.0]
    items = rm.featurize([rc.generate_complex(0)], rm.VoxelHeadConfig(), rm.GraphHeadConfig())
    assert sc([harness.PoseRecord("c", "t", 0, (items[0].grid, items[0].graph))]) == [1.0]
    assert calls == [("raw", 3), ("pairs", 1)]


def test_unscorable_pose_raises_like_reference():
    class Fake:
        def predict_batch(self, items):
            return [None], [(0, "voxel grid contains non-finite values")]
    with pytest.raises(ValueError, match="unscorable pose c/t/0: voxel grid contains non-finite values"):
        harness.ModelScorer(Fake())([harness.PoseRecord("c", "t", 0, ("g", "h"))])


def test_reference_checkpoint_with_optimizer_roundtrips(tmp_path):
    rc, rm, ck = _ref()
    from fusionscreen import optim
    ref = rm.FusionModel(rm.VoxelHeadConfig(), rm.GraphHeadConfig(), rm.table_coherent_fusion_config(), seed=5)
    opt = optim.Optimizer(optim.OptimizerConfig("adam", 1e-3))
    grads = {k: np.ones_like(v) for k, v in ref.all_params().items()}
    params = {k: v.copy() for k, v in ref.all_params().items()}
    opt.step(params, grads)
    path = tmp_path / "ref.npz"
    ref.save(path, opt)
    from paper_2104_04547_b200.checkpoint import load_checkpoint, save_checkpoint
    p, o, meta = load_checkpoint(path)
    wp, wo, wmeta = ck.load_checkpoint(path)
    assert meta == wmeta and sorted(p) == sorted(wp)
    assert all(np.array_equal(p[k], wp[k]) for k in p)
    assert o.step_count == wo.step_count and o.kind == wo.cfg.kind
    for k, v in wo.state_arrays().items():
        assert np.array_equal(o.arrays[k], v)
    # written back by this package, the reference reads the same state
    path2 = tmp_path / "back.npz"
    save_checkpoint(path2, p, o, meta)
    p2, o2, meta2 = ck.load_checkpoint(path2)
    assert meta2 == meta and o2.step_count == o.step_count
    assert all(np.array_equal(p2[k], p[k]) for k in p)
    back = models.FusionModel.load(path)
    assert np.array_equal(back.voxel_params["conv1_w"], ref.voxel_params["conv1_w"])


def test_load_checkpoint_returns_three_tuple(tmp_path):
    m = _model()
    m.save(tmp_path / "m.npz")
    from paper_2104_04547_b200.checkpoint import load_checkpoint
    params, opt, meta = load_checkpoint(tmp_path / "m.npz")
    assert opt is None and meta["model"] == "fusion" and len(params) == len(m.all_params())


def test_param_shapes_checked_before_packing():
    m = _model()
    flat = m.all_params()
    models.check_param_shapes(m.voxel_cfg, m.graph_cfg, m.fusion_cfg, flat)
    bad = dict(flat)
    bad["voxel/conv2_w"] = np.zeros((3, 3))
    with pytest.raises(ValueError, match="conv2_w"):
        models.check_param_shapes(m.voxel_cfg, m.graph_cfg, m.fusion_cfg, bad)
    missing = dict(flat)
    del missing["fusion/fuse0_w"]
    with pytest.raises(ValueError, match="missing"):
        models.check_param_shapes(m.voxel_cfg, m.graph_cfg, m.fusion_cfg, missing)


def test_device_model_cache_is_identity_based(monkeypatch):
    """No per-call hashing of the 808k parameters: the packed model is reused
    until a parameter is rebound, set_params() runs or invalidate() is called."""
    from paper_2104_04547_b200 import engine
    built = []

    class FakeDM:
        def __init__(self, *a, **k):
            built.append(1)
    monkeypatch.setattr(engine, "DeviceModel", FakeDM)
    m = _model()
    a = m.device_model()
    assert m.device_model() is a and len(built) == 1
    m.voxel_params["conv1_w"] = m.voxel_params["conv1_w"].copy()
    b = m.device_model()
    assert b is not a and len(built) == 2
    m.set_params({"graph/embed_b": np.zeros(24)})
    m.device_model()
    assert len(built) == 3
    m.invalidate()
    m.device_model()
    assert len(built) == 4
