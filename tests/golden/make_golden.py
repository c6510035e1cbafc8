"""Generate golden vectors by running the UNMODIFIED reference (fusionscreen).

Run in the build container only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The outputs (``*.npz`` next to this file) are committed; the GPU box never
reads /root/reference.  Every array here comes from a reference call:
``generate_complex`` (complexes.py:102), ``voxelize`` (:171), ``build_graph``
(:223), ``FusionModel`` (models.py:412) / ``predict_batch`` (:470),
``voxel_head_forward`` / ``graph_head_forward`` (:590-614).
"""

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from fusionscreen import complexes, harness, models  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
BASELINE_GEN = complexes.GenParams(n_protein=(1000, 1000), n_ligand=(64, 64))


def params_digest(params):
    h = hashlib.sha256()
    for k in sorted(params):
        h.update(k.encode())
        h.update(np.ascontiguousarray(params[k], dtype=np.float64).tobytes())
    return h.hexdigest()


def pack_complex(cs):
    off = np.cumsum([0] + [c.n_atoms for c in cs]).astype(np.int64)
    return dict(atom_off=off,
                positions=np.concatenate([c.positions for c in cs]),
                elements=np.concatenate([c.elements for c in cs]).astype(np.int64),
                roles=np.concatenate([c.roles for c in cs]).astype(np.int64))


def edge_cases():
    """Hand-made complexes covering the reference's known-answer tests
    (test_complexes.py:95-206) plus boundary geometry."""
    out = []
    base = complexes.generate_complex(0, complexes.GenParams(c_elem=4))

    def mk(pos, roles, elems, cid):
        return complexes.SyntheticComplex(cid, np.asarray(pos, dtype=np.float64),
                                          np.asarray(elems, dtype=np.int64),
                                          np.asarray(roles, dtype=np.int64), 0.0)
    # out-of-box atoms clip to boundary voxels; huge element clips to c_elem-1
    out.append(mk([[99.0, 99.0, 99.0], [-99.0, 0.0, 7.999], [8.0, -8.0, 0.0],
                   [0.0, 0.0, 0.0], [1.5, 0.0, 0.0]],
                  [0, 1, 0, 1, 1], [0, 7, -3, 2, 1], "edge-clip"))
    # exact-threshold distances along the axes (d == 2.24 and d == 5.22)
    out.append(mk([[0, 0, 0], [2.24, 0, 0], [0, 5.22, 0], [0, 0, 6.0],
                   [1.0, 1.0, 1.0]],
                  [1, 1, 0, 0, 1], [0, 1, 2, 3, 0], "edge-thresh"))
    # coincident atoms (d == 0) and a dense clump
    rng = np.random.default_rng(5)
    clump = np.vstack([np.zeros((6, 3)), rng.normal(0, 0.7, size=(40, 3))])
    out.append(mk(clump, rng.integers(0, 2, len(clump)), rng.integers(0, 4, len(clump)),
                  "edge-clump"))
    del base
    return out


def graph_edge_cases():
    """Complexes that drive every special path of the GPU radius graphs
    (graph_csr.cu / featurize.cu): threshold-exact and +-1-ulp distances in
    several directions, a ligand larger than the 64-atom bitmask path, a
    larger ligand than pocket (smaller role = protein), coordinates beyond the
    1024 A fp32 prefilter bound, a compressed pocket with > 96 covalent
    candidates per row, coincident atoms and single-atom / single-role poses."""
    rng = np.random.default_rng(11)
    out = []

    def mk(pos, roles, elems, cid):
        return complexes.SyntheticComplex(cid, np.asarray(pos, dtype=np.float64),
                                          np.asarray(elems, dtype=np.int64),
                                          np.asarray(roles, dtype=np.int64), 0.0)
    # +-1 ulp around both thresholds along axes and diagonals
    pos, roles = [], []
    for k, (t, same) in enumerate(((2.24, True), (5.22, False))):
        for d_i, direc in enumerate(([1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 0], [1, 1, 1], [3, -4, 12])):
            u = np.asarray(direc, dtype=np.float64) / np.linalg.norm(direc)
            for j, dist in enumerate((np.nextafter(t, 0), t, np.nextafter(t, 10))):
                c = np.array([-6.0 + 3.0 * d_i, -6.0 + 4.0 * j, -6.0 + 6.0 * k])
                pos += [c, c + dist * u]
                roles += [0, 0 if same else 1]
    out.append(mk(pos, roles, rng.integers(0, 4, len(pos)), "edge-ulp"))
    # ligand > 64 atoms (bitmask non-covalent path off), pocket 300
    p = rng.uniform(-8, 8, (300, 3))
    lig = np.clip(rng.normal(0, 2.0, (100, 3)), -8, 8)
    out.append(mk(np.vstack([p, lig]), [0] * 300 + [1] * 100, rng.integers(0, 4, 400), "edge-biglig"))
    # more ligand than protein atoms (smaller role = protein)
    p = rng.uniform(-8, 8, (40, 3))
    lig = np.clip(rng.normal(0, 2.5, (90, 3)), -8, 8)
    out.append(mk(np.vstack([p, lig]), [0] * 40 + [1] * 90, rng.integers(0, 4, 130), "edge-swap"))
    # far from the origin: |coords| >= 1024 A (fp32 prefilter disabled)
    p = rng.uniform(-8, 8, (200, 3)) + 2048.0
    lig = rng.normal(2048.0, 1.8, (40, 3))
    out.append(mk(np.vstack([p, lig]), [0] * 200 + [1] * 40, rng.integers(0, 4, 240), "edge-far"))
    # compressed pocket: 400 atoms in a 5 A cube (> 96 candidates per covalent row)
    p = rng.uniform(-2.5, 2.5, (400, 3))
    lig = rng.uniform(-3.0, 3.0, (30, 3))
    out.append(mk(np.vstack([p, lig]), [0] * 400 + [1] * 30, rng.integers(0, 4, 430), "edge-dense"))
    # coincident atoms of both roles, a lone atom, a protein-only complex
    c = np.zeros((8, 3))
    out.append(mk(c, [0, 1] * 4, [0, 1, 2, 3] * 2, "edge-coincident"))
    out.append(mk([[1.0, 2.0, 3.0]], [1], [2], "edge-single"))
    out.append(mk(rng.uniform(-8, 8, (120, 3)), [0] * 120, rng.integers(0, 4, 120), "edge-protein-only"))
    return out


def write_graph_edge_golden():
    cs = graph_edge_cases()
    cov_e, cov_d, ncov_e, ncov_d, feats = [], [], [], [], []
    cov_off, ncov_off = [0], [0]
    for c in cs:
        g = complexes.build_graph(c, 2.24, 5.22, 4, 16.0)
        feats.append(g.node_features)
        cov_e.append(g.covalent_edges.astype(np.int32).reshape(-1, 2))
        cov_d.append(g.covalent_dists)
        ncov_e.append(g.noncovalent_edges.astype(np.int32).reshape(-1, 2))
        ncov_d.append(g.noncovalent_dists)
        cov_off.append(cov_off[-1] + len(g.covalent_edges))
        ncov_off.append(ncov_off[-1] + len(g.noncovalent_edges))
    np.savez_compressed(
        os.path.join(HERE, "graph_edge_golden.npz"), **pack_complex(cs),
        names=np.array([c.complex_id for c in cs]),
        node_features=np.concatenate(feats),
        cov_edges=np.concatenate(cov_e), cov_dists=np.concatenate(cov_d),
        ncov_edges=np.concatenate(ncov_e), ncov_dists=np.concatenate(ncov_d),
        cov_off=np.asarray(cov_off, dtype=np.int64), ncov_off=np.asarray(ncov_off, dtype=np.int64))


def write_campaign_golden():
    """run_campaign (harness.py:348-424) with the reference ModelScorer over a
    small featurized library, with record corruption and job failures, so the
    B200 scorer + campaign driver can be replayed record for record."""
    import json
    import tempfile
    vcfg, gcfg = models.VoxelHeadConfig(), models.GraphHeadConfig()
    model = models.FusionModel(vcfg, gcfg, models.table_coherent_fusion_config(), seed=0)
    cs = [complexes.generate_complex(5000 + s) for s in range(30)]
    items = models.featurize(cs, vcfg, gcfg)
    lib = [harness.PoseRecord(f"c{i // 3:03d}", "t0" if i % 2 else "t1", i % 3, (it.grid, it.graph))
           for i, it in enumerate(items)]
    plan = harness.FaultPlan(record_corruption_rate=0.15, job_failure_rate=0.3, seed=4)
    with tempfile.TemporaryDirectory() as d:
        preds, rep = harness.run_campaign(lib, harness.ModelScorer(model), n_jobs=3, plan=plan, out_dir=d,
                                          parallelism=2, retries=3, ranks_per_job=2, batch_size=4)
        shards = {}
        for name in sorted(os.listdir(d)):
            if name.endswith(".jsonl") or (name.endswith(".json") and name != harness.MANIFEST_NAME):
                shards[name] = open(os.path.join(d, name)).read()
        manifest = json.load(open(os.path.join(d, harness.MANIFEST_NAME)))
    manifest.pop("timings")
    rows = [(r.compound_id, r.target_id, r.pose_id, r.job_id, r.rank_id) for r in preds]
    np.savez_compressed(
        os.path.join(HERE, "campaign_golden.npz"), **pack_complex(cs),
        pred_rows=np.array(json.dumps(rows)), pred_scores=np.array([r.predicted_pk for r in preds]),
        corrupted=np.array(json.dumps(rep.corrupted)), manifest=np.array(json.dumps(manifest, sort_keys=True)),
        files=np.array(json.dumps(shards, sort_keys=True)))


def main():
    # ---- featurizer golden: default-distribution + BASELINE-shape + edge cases
    cs = [complexes.generate_complex(s) for s in range(6)]
    cs += [complexes.generate_complex(1000 + s, BASELINE_GEN) for s in range(2)]
    cs += edge_cases()
    grid_cfg = complexes.GridConfig(extent=16, c_elem=4, box_size=16.0)
    vox_nz_idx, vox_nz_val, vox_off = [], [], [0]
    feats, cov_e, cov_d, ncov_e, ncov_d = [], [], [], [], []
    cov_off, ncov_off = [0], [0]
    for c in cs:
        occ = complexes.voxelize(c, grid_cfg).occupancy
        nz = np.flatnonzero(occ)
        vox_nz_idx.append(nz.astype(np.int32))
        vox_nz_val.append(occ.reshape(-1)[nz])
        vox_off.append(vox_off[-1] + len(nz))
        g = complexes.build_graph(c, 2.24, 5.22, 4, 16.0)
        feats.append(g.node_features)
        # reference order is kd-tree traversal order; store as emitted
        cov_e.append(g.covalent_edges.astype(np.int32).reshape(-1, 2))
        cov_d.append(g.covalent_dists)
        ncov_e.append(g.noncovalent_edges.astype(np.int32).reshape(-1, 2))
        ncov_d.append(g.noncovalent_dists)
        cov_off.append(cov_off[-1] + len(g.covalent_edges))
        ncov_off.append(ncov_off[-1] + len(g.noncovalent_edges))
    np.savez_compressed(
        os.path.join(HERE, "featurize_golden.npz"),
        **pack_complex(cs),
        vox_nz_idx=np.concatenate(vox_nz_idx), vox_nz_val=np.concatenate(vox_nz_val),
        vox_off=np.asarray(vox_off, dtype=np.int64),
        node_features=np.concatenate(feats),
        cov_edges=np.concatenate(cov_e), cov_dists=np.concatenate(cov_d),
        ncov_edges=np.concatenate(ncov_e), ncov_dists=np.concatenate(ncov_d),
        cov_off=np.asarray(cov_off, dtype=np.int64),
        ncov_off=np.asarray(ncov_off, dtype=np.int64))

    # ---- model golden: default Coherent Fusion model, seed 0, BASELINE shape
    vcfg, gcfg = models.VoxelHeadConfig(), models.GraphHeadConfig()
    fcfg = models.table_coherent_fusion_config()
    model = models.FusionModel(vcfg, gcfg, fcfg, seed=0)
    poses = [complexes.generate_complex(2000 + s, BASELINE_GEN) for s in range(4)]
    poses += [complexes.generate_complex(3000 + s) for s in range(2)]
    items = models.featurize(poses, vcfg, gcfg)
    pairs = [(it.grid, it.graph) for it in items]
    preds, errors = model.predict_batch(pairs)
    assert not errors
    pv, lat_v = models.voxel_head_forward(model.voxel_params, vcfg, [it.grid for it in items])
    pg, lat_g = models.graph_head_forward(model.graph_params, gcfg, [it.graph for it in items])
    late = models.FusionModel(vcfg, gcfg, models.FusionConfig(mode="late"), seed=0)
    late_preds, _ = late.predict_batch(pairs)
    mid = models.FusionModel(vcfg, gcfg, models.table_mid_fusion_config(), seed=3)
    mid_preds, _ = mid.predict_batch(pairs)
    np.savez_compressed(
        os.path.join(HERE, "model_golden.npz"), **pack_complex(poses),
        scores=np.asarray(preds), pred_v=pv, lat_v=lat_v, pred_g=pg, lat_g=lat_g,
        late_scores=np.asarray(late_preds), mid_scores=np.asarray(mid_preds),
        params_sha256=np.frombuffer(params_digest(model.all_params()).encode(), dtype=np.uint8),
        mid_params_sha256=np.frombuffer(params_digest(mid.all_params()).encode(), dtype=np.uint8))

    # ---- toy-config golden (the reference's own test fixtures, conftest.py:7-49)
    tv = models.VoxelHeadConfig(grid_extent=8, in_channels=2, conv_filters_1=2,
                                conv_filters_2=2, dense_nodes=8, kernel_1=3,
                                dropout_early=0.0, dropout_mid=0.0)
    tg = models.GraphHeadConfig(c_elem=1, k_cov=2, k_noncov=2, gather_width_cov=4,
                                gather_width_noncov=4)
    tf = models.FusionConfig(mode="coherent", n_fusion_layers=3, fusion_dense_nodes=6,
                             dropout_early=0.0, dropout_mid=0.0, dropout_late=0.0)
    tgen = complexes.GenParams(box_size=8.0, c_elem=1, n_protein=(8, 12), n_ligand=(3, 5),
                               noise_sigma=0.05)
    tcs = [complexes.generate_complex(i, tgen) for i in range(16)]
    titems = models.featurize(tcs, tv, tg, box_size=8.0)
    tmodel = models.FusionModel(tv, tg, tf, seed=0)
    tpreds, _ = tmodel.predict_batch([(it.grid, it.graph) for it in titems])
    np.savez_compressed(os.path.join(HERE, "toy_golden.npz"), **pack_complex(tcs),
                        scores=np.asarray(tpreds))
    write_graph_edge_golden()
    write_campaign_golden()
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
