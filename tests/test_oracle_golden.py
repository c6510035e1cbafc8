"""Pin the CPU oracle against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import fusion_oracle as orc
from tests._cfg import (COHERENT, GRAPH, LATE, MID, TOY_FUSION, TOY_GRAPH, TOY_VOXEL,
                        VOXEL, complexes_of, load)


def _digest(*dicts, prefixes=("voxel", "graph", "fusion")):
    flat = {}
    for pre, d in zip(prefixes, dicts):
        for k, v in d.items():
            flat[f"{pre}/{k}"] = v
    h = hashlib.sha256()
    for k in sorted(flat):
        h.update(k.encode())
        h.update(np.ascontiguousarray(flat[k], dtype=np.float64).tobytes())
    return h.hexdigest()


def test_voxelize_matches_reference_bitwise():
    z = load("featurize_golden.npz")
    for p, (pos, el, ro) in enumerate(complexes_of(z)):
        occ = orc.voxelize(pos, el, ro, 16, 4, 16.0).reshape(-1)
        s, e = z["vox_off"][p], z["vox_off"][p + 1]
        want = np.zeros_like(occ)
        want[z["vox_nz_idx"][s:e]] = z["vox_nz_val"][s:e]
        assert np.array_equal(occ, want), p
        assert occ.sum() == len(pos)


def test_build_graph_matches_reference_bitwise():
    z = load("featurize_golden.npz")
    noff = z["atom_off"]
    for p, (pos, el, ro) in enumerate(complexes_of(z)):
        f = orc.node_features(pos, el, ro, 4, 16.0)
        assert np.array_equal(f, z["node_features"][noff[p]:noff[p + 1]])
        ce, cd, ne, nd = orc.radius_pairs(pos, ro, 2.24, 5.22)
        for edges, dists, key in ((ce, cd, "cov"), (ne, nd, "ncov")):
            s, e = z[f"{key}_off"][p], z[f"{key}_off"][p + 1]
            we, wd = orc.canonical_edges(z[f"{key}_edges"][s:e], z[f"{key}_dists"][s:e])
            assert np.array_equal(edges, we), (p, key)
            assert np.array_equal(dists, wd), (p, key)   # float64 bitwise


def test_threshold_range_enforced():
    with pytest.raises(ValueError):
        orc.radius_pairs(np.zeros((2, 3)), [0, 1], 1.1, 5.22)
    with pytest.raises(ValueError):
        orc.radius_pairs(np.zeros((2, 3)), [0, 1], 2.24, 6.0)


def test_param_init_matches_reference():
    z = load("model_golden.npz")
    v, g, f = orc.init_params(VOXEL, GRAPH, COHERENT, seed=0)
    assert _digest(v, g, f) == bytes(z["params_sha256"]).decode()
    v, g, f = orc.init_params(VOXEL, GRAPH, MID, seed=3)
    assert _digest(v, g, f) == bytes(z["mid_params_sha256"]).decode()


def _score_all(z, vcfg, gcfg, fcfg, seed, box=16.0):
    params = orc.init_params(vcfg, gcfg, fcfg, seed)
    return [orc.score_pose(params, (vcfg, gcfg, fcfg), pos, el, ro, box)
            for pos, el, ro in complexes_of(z)]


def test_coherent_scores_and_latents_match_reference():
    z = load("model_golden.npz")
    outs = _score_all(z, VOXEL, GRAPH, COHERENT, 0)
    np.testing.assert_allclose([o["score"] for o in outs], z["scores"], rtol=1e-12)
    np.testing.assert_allclose(np.stack([o["lat_v"] for o in outs]), z["lat_v"],
                               rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(np.stack([o["lat_g"] for o in outs]), z["lat_g"],
                               rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose([o["pred_v"] for o in outs], z["pred_v"], rtol=1e-12)
    np.testing.assert_allclose([o["pred_g"] for o in outs], z["pred_g"], rtol=1e-12)


def test_late_and_mid_modes_match_reference():
    z = load("model_golden.npz")
    late = _score_all(z, VOXEL, GRAPH, LATE, 0)
    np.testing.assert_allclose([o["score"] for o in late], z["late_scores"], rtol=1e-12)
    mid = _score_all(z, VOXEL, GRAPH, MID, 3)
    np.testing.assert_allclose([o["score"] for o in mid], z["mid_scores"], rtol=1e-12)


def test_toy_config_matches_reference():
    z = load("toy_golden.npz")
    outs = _score_all(z, TOY_VOXEL, TOY_GRAPH, TOY_FUSION, 0, box=8.0)
    np.testing.assert_allclose([o["score"] for o in outs], z["scores"], rtol=1e-12)


def test_topk_tie_rule():
    s = np.array([0.5, 0.7, 0.7, 0.1, 0.7])
    vals, idx = orc.topk(s, 3, index_base=10)
    assert idx.tolist() == [11, 12, 14]
    best = orc.best_pose(["a", "a", "b"], ["t", "t", "t"], [3, 1, 0], [1.0, 1.0, 2.0])
    assert best[("a", "t")] == (1, 1.0)


def _c_radius(z):
    from oracle import radius_c
    return radius_c.radius_pairs_batch(z["positions"], z["roles"], z["atom_off"], 2.24, 5.22)


def test_c_radius_oracle_matches_reference_bitwise():
    """oracle/radius_graph.c (the checker the GPU edge tests use at scale) is
    pinned against the reference's build_graph on every golden complex,
    including the +-1-ulp, far-from-origin, dense and single-role cases."""
    for name in ("featurize_golden.npz", "graph_edge_golden.npz"):
        z = load(name)
        ce, cd, coff, ne, nd, noff = _c_radius(z)
        for p in range(len(z["atom_off"]) - 1):
            for edges, dists, off, key in ((ce, cd, coff, "cov"), (ne, nd, noff, "ncov")):
                s, e = z[f"{key}_off"][p], z[f"{key}_off"][p + 1]
                we, wd = orc.canonical_edges(z[f"{key}_edges"][s:e], z[f"{key}_dists"][s:e])
                assert np.array_equal(edges[off[p]:off[p + 1]], we), (name, p, key)
                assert np.array_equal(dists[off[p]:off[p + 1]], wd), (name, p, key)


def test_c_radius_oracle_matches_numpy_oracle():
    from oracle import radius_c
    from paper_2104_04547_b200 import synth
    pk = synth.make_pocket(1000, seed=0)
    lib = synth.make_poses(2, 2, seed=9)
    for p in range(lib.n_poses):
        pos, _, ro = synth.complex_arrays(pk, lib, p)
        for a, b in zip(orc.radius_pairs(pos, ro), radius_c.radius_pairs(pos, ro)):
            assert np.array_equal(a, b)


def test_config1_oracle_fixture_matches_oracle():
    """tests/golden/config1_oracle.npz (scores the GPU config-1 test compares
    against) is the pinned oracle's output: spot-check 3 of its poses."""
    from paper_2104_04547_b200 import synth
    z = load("config1_oracle.npz")
    pocket = synth.make_pocket(1000, seed=0)
    lib = synth.make_poses(103, 10, seed=1, ligand_atoms=(16, 64)).slice(0, 1024)
    params = orc.init_params(VOXEL, GRAPH, COHERENT, 0)
    for p in (0, 511, 1023):
        s = orc.score_pose(params, (VOXEL, GRAPH, COHERENT), *synth.complex_arrays(pocket, lib, p))["score"]
        assert abs(s - z["scores"][p]) <= 1e-12 * abs(s)    # BLAS thread count changes the last ulp
