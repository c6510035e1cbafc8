"""Host-side logic of the package (configs, init, checkpoints, sharding,
synthetic libraries) -- CPU only.  Mirrors the reference tests
(test_models.py:23-83, test_harness.py, test_checkpoint.py)."""

import numpy as np
import pytest

from oracle import fusion_oracle as orc
from paper_2104_04547_b200 import complexes as cx
from paper_2104_04547_b200 import harness, models, synth
from paper_2104_04547_b200.models import (FusionConfig, GraphHeadConfig, VoxelHeadConfig,
                                          table_coherent_fusion_config, table_mid_fusion_config)
from tests._cfg import COHERENT, GRAPH, MID, VOXEL, load


def test_config_validation_matches_reference():
    for bad in (1, 9):
        with pytest.raises(ValueError):
            GraphHeadConfig(k_cov=bad)
        with pytest.raises(ValueError):
            GraphHeadConfig(k_noncov=bad)
    assert GraphHeadConfig(gather_width_noncov=128).dense_widths == (85, 42)
    assert GraphHeadConfig(gather_width_noncov=24).dense_widths == (16, 8)
    assert VoxelHeadConfig(grid_extent=16, conv_filters_2=64).flat_width == 64 * 4 ** 3
    with pytest.raises(ValueError):
        FusionConfig(mode="early")
    for bad in (2, 6):
        with pytest.raises(ValueError):
            FusionConfig(mode="coherent", n_fusion_layers=bad)
    FusionConfig(mode="late", n_fusion_layers=2)
    c = table_coherent_fusion_config()
    assert (c.mode, c.n_fusion_layers, c.batch_size, c.pre_trained) == ("coherent", 4, 48, True)
    assert c.optimizer.learning_rate == pytest.approx(1.08e-4)
    m = table_mid_fusion_config()
    assert (m.mode, m.n_fusion_layers, m.model_specific_layers) == ("mid", 5, True)


def test_fusion_model_params_equal_reference_init():
    z = load("model_golden.npz")
    model = models.FusionModel(VoxelHeadConfig(), GraphHeadConfig(), table_coherent_fusion_config(), seed=0)
    v, g, f = orc.init_params(VOXEL, GRAPH, COHERENT, seed=0)
    flat = model.all_params()
    for pre, d in (("voxel", v), ("graph", g), ("fusion", f)):
        for k, arr in d.items():
            assert np.array_equal(flat[f"{pre}/{k}"], arr), k
    assert len(flat) == len(v) + len(g) + len(f)
    assert sum(a.size for a in flat.values()) == 808_646
    # digest pinned against the reference itself
    from tests.test_oracle_golden import _digest
    assert _digest(v, g, f) == bytes(z["params_sha256"]).decode()
    mid = models.FusionModel(VoxelHeadConfig(), GraphHeadConfig(), table_mid_fusion_config(), seed=3)
    v, g, f = orc.init_params(VOXEL, GRAPH, MID, seed=3)
    assert np.array_equal(mid.fusion_params["fuse4_w"], f["fuse4_w"])


def test_checkpoint_roundtrip_bitwise(tmp_path):
    m = models.FusionModel(VoxelHeadConfig(), GraphHeadConfig(), table_mid_fusion_config(), seed=7)
    p = tmp_path / "m.npz"
    m.save(p)
    back = models.FusionModel.load(p)
    assert back.voxel_cfg == m.voxel_cfg and back.graph_cfg == m.graph_cfg
    assert back.fusion_cfg == m.fusion_cfg
    for k, v in m.all_params().items():
        assert np.array_equal(back.all_params()[k], v)


def test_reference_checkpoint_loads(tmp_path):
    """A checkpoint written by the reference's own save_checkpoint format
    (checkpoint.py:21-45, with optimizer state) loads unchanged."""
    import json
    m = models.FusionModel(VoxelHeadConfig(), GraphHeadConfig(), table_coherent_fusion_config(), seed=1)
    payload = {f"param/{k}": v for k, v in m.all_params().items()}
    payload["opt/voxel/conv1_w::m"] = np.zeros(3)
    header = {"format_version": 1, "param_names": sorted(m.all_params()),
              "meta": {"model": "fusion", "voxel_cfg": vars(m.voxel_cfg) | {},
                       "graph_cfg": vars(m.graph_cfg) | {},
                       "fusion_cfg": models._fusion_cfg_dict(m.fusion_cfg), "seed": 1},
              "optimizer": {"kind": "adam", "learning_rate": 1e-3, "coefficients": {}, "step_count": 2}}
    payload["__header__"] = np.frombuffer(json.dumps(header, sort_keys=True).encode(), dtype=np.uint8)
    path = tmp_path / "ref.npz"
    with open(path, "wb") as fh:
        np.savez(fh, **payload)
    back = models.FusionModel.load(path)
    assert np.array_equal(back.voxel_params["conv4_w"], m.voxel_params["conv4_w"])


def test_generate_complex_matches_reference_golden():
    z = load("featurize_golden.npz")
    for s in range(6):
        c = cx.generate_complex(s)
        a, b = z["atom_off"][s], z["atom_off"][s + 1]
        assert np.array_equal(c.positions, z["positions"][a:b])
        assert np.array_equal(c.elements, z["elements"][a:b])
        assert np.array_equal(c.roles, z["roles"][a:b])


def test_balanced_and_compound_aligned_shards():
    assert harness.balanced_sizes(10, 3) == [4, 3, 3]
    with pytest.raises(ValueError):
        harness.balanced_sizes(3, 0)
    lib = synth.make_poses(37, poses_per_compound=10, seed=2)
    for parts in (1, 2, 3, 8):
        b = harness.compound_aligned_bounds(lib.compound, parts)
        assert b[0][0] == 0 and b[-1][1] == lib.n_poses
        for (s0, e0), (s1, e1) in zip(b, b[1:]):
            assert e0 == s1
        for s, e in b:
            if 0 < s < lib.n_poses:
                assert lib.compound[s] != lib.compound[s - 1]   # never splits a compound
        sizes = [len(set(lib.compound[s:e])) for s, e in b]
        assert max(sizes) - min(sizes) <= 1


def test_synthetic_library_distribution():
    pocket = synth.make_pocket(1000, seed=0)
    assert pocket.xyz.shape == (1000, 3) and np.all(np.abs(pocket.xyz) <= 8.0)
    lib = synth.make_poses(200, poses_per_compound=10, seed=1)
    sizes = np.diff(lib.atom_off)
    assert sizes.min() >= 16 and sizes.max() <= 64
    assert np.all(np.abs(lib.xyz) <= 8.0) and np.all(lib.role == 1)
    # all poses of a compound share the element list
    a0, a1 = lib.atom_off[0], lib.atom_off[1]
    b0, b1 = lib.atom_off[1], lib.atom_off[2]
    assert np.array_equal(lib.elem[a0:a1], lib.elem[b0:b1])
    # centres ~U[-2, 2): ligand means stay near the pocket centre
    means = np.array([lib.xyz[lib.atom_off[p]:lib.atom_off[p + 1]].mean(0) for p in range(50)])
    assert np.all(np.abs(means) < 4.0)
    part = lib.slice(10, 20)
    assert part.n_poses == 10 and part.atom_off[0] == 0
    pos, el, ro = synth.complex_arrays(pocket, lib, 3)
    assert len(pos) == 1000 + sizes[3] and ro[:1000].sum() == 0 and ro[1000:].min() == 1


def test_pack_graphs_lifts_edges_to_global_ids():
    g1 = cx.ComplexGraph(np.zeros((3, 8)), np.array([[0, 1]]), np.zeros((0, 2), int), np.ones(1), np.zeros(0))
    g2 = cx.ComplexGraph(np.zeros((2, 8)), np.array([[0, 1]]), np.array([[0, 1]]), np.ones(1), np.ones(1))
    feats, off, ce, ne = models._pack_graphs([g1, g2])
    assert off.tolist() == [0, 3, 5]
    assert ce.tolist() == [[0, 1], [3, 4]] and ne.tolist() == [[3, 4]]
    bad = cx.ComplexGraph(np.zeros((2, 8)), np.array([[0, 5]]), np.zeros((0, 2), int), np.ones(1), np.zeros(0))
    with pytest.raises(ValueError):
        models._pack_graphs([bad])


def test_validate_item_reason_strings():
    m = models.FusionModel(VoxelHeadConfig(), GraphHeadConfig(), table_coherent_fusion_config())
    assert m._validate_item("x") == "item is not a (VoxelGrid, ComplexGraph) pair"
    assert m._validate_item((1, 2)) == "item is not a (VoxelGrid, ComplexGraph) pair"
    g = cx.ComplexGraph(np.zeros((2, 8)), np.zeros((0, 2), int), np.zeros((0, 2), int), np.zeros(0), np.zeros(0))
    r = m._validate_item((cx.VoxelGrid(np.zeros((2, 4, 4, 4))), g))
    assert "shape" in r
    r = m._validate_item((cx.VoxelGrid(np.zeros((8, 16, 16, 16))),
                          cx.ComplexGraph(np.zeros((2, 5)), g.covalent_edges, g.noncovalent_edges,
                                          g.covalent_dists, g.noncovalent_dists)))
    assert r.startswith("graph feature width")


def test_fusion_model_pickles_and_deep_copies():
    """Campaign drivers may copy or pickle the model (the packed device model
    and its lock are rebuilt lazily, never serialised)."""
    import copy
    import pickle

    from paper_2104_04547_b200 import models
    m = models.FusionModel(models.VoxelHeadConfig(), models.GraphHeadConfig(),
                           models.table_coherent_fusion_config(), seed=0)
    for m2 in (copy.deepcopy(m), pickle.loads(pickle.dumps(m))):
        assert m2._dev is None
        assert m2._dev_lock is not None
        for k, v in m.all_params().items():
            assert np.array_equal(v, m2.all_params()[k])
