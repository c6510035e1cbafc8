"""The campaign caller of the scoring path (harness.run_job / run_campaign,
restating /root/reference/pkg/src/fusionscreen/harness.py:245-424) replayed
against the reference's own golden run (tests/golden/campaign_golden.npz,
made by make_golden.py with the reference ModelScorer, record corruption and
job failures).  CPU: the driver semantics with the golden scores; GPU: the
B200 ModelScorer behind it, scores within 1e-3 of the reference."""

import json
import os

import numpy as np
import pytest

from paper_2104_04547_b200 import harness
from tests._cfg import complexes_of, load


def _reference(module):
    """The unmodified reference module, where it exists (build container only)."""
    import importlib
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not present (GPU box)")
    if src not in sys.path:
        sys.path.append(src)
    return importlib.import_module(f"fusionscreen.{module}")


def _golden():
    z = load("campaign_golden.npz")
    rows = [tuple(r) for r in json.loads(str(z["pred_rows"]))]
    return z, rows, json.loads(str(z["corrupted"])), json.loads(str(z["manifest"])), json.loads(str(z["files"]))


def _library(payloads):
    # same keys as make_golden.write_campaign_golden
    return [harness.PoseRecord(f"c{i // 3:03d}", "t0" if i % 2 else "t1", i % 3, pl) for i, pl in enumerate(payloads)]


def _run(tmp_path, scorer, payloads):
    plan = harness.FaultPlan(record_corruption_rate=0.15, job_failure_rate=0.3, seed=4)
    preds, rep = harness.run_campaign(_library(payloads), scorer, n_jobs=3, plan=plan, out_dir=tmp_path,
                                      parallelism=2, retries=3, ranks_per_job=2, batch_size=4)
    files = {n: open(os.path.join(tmp_path, n)).read() for n in sorted(os.listdir(tmp_path))
             if n.endswith(".jsonl") or (n.endswith(".json") and n != harness.MANIFEST_NAME)}
    manifest = json.load(open(os.path.join(tmp_path, harness.MANIFEST_NAME)))
    manifest.pop("timings")
    return preds, rep, files, manifest


def _check(preds, rep, files, manifest, scores_close):
    z, rows, corrupted, want_manifest, want_files = _golden()
    assert [(r.compound_id, r.target_id, r.pose_id, r.job_id, r.rank_id) for r in preds] == rows
    assert [list(c) for c in rep.corrupted] == corrupted
    assert json.loads(json.dumps(manifest, sort_keys=True)) == want_manifest
    scores_close(np.array([r.predicted_pk for r in preds]), z["pred_scores"])
    assert sorted(files) == sorted(want_files)
    for name, text in files.items():
        if name.startswith("shard_"):
            got = [json.loads(x) for x in text.splitlines()]
            want = [json.loads(x) for x in want_files[name].splitlines()]
            assert [{k: v for k, v in r.items() if k != "predicted_pk"} for r in got] == \
                [{k: v for k, v in r.items() if k != "predicted_pk"} for r in want], name
            scores_close(np.array([r["predicted_pk"] for r in got]), np.array([r["predicted_pk"] for r in want]))
        else:
            assert text == want_files[name], name


def test_campaign_driver_replays_reference_with_golden_scores(tmp_path):
    """Driver semantics alone: a scorer returning the reference's scores must
    reproduce the reference campaign byte for byte (shards, manifests,
    corrupted list, exactly-once retries)."""
    z, rows, *_ = _golden()
    by_key = {(r[0], r[1], r[2]): s for r, s in zip(rows, z["pred_scores"])}

    def scorer(batch):
        return [float(by_key[(p.compound_id, p.target_id, p.pose_id)]) for p in batch]

    out = _run(tmp_path, scorer, [None] * 30)
    _check(*out, lambda a, b: np.testing.assert_array_equal(a, b))


def test_campaign_driver_matches_reference_synthetic_scorer(tmp_path):
    """Where the reference is importable (build container): its run_campaign and
    ours give identical records with its SyntheticScorer."""
    ref = _reference("harness")
    lib_ref = [ref.PoseRecord(f"c{i // 7}", "t", i % 7) for i in range(61)]
    lib_own = [harness.PoseRecord(f"c{i // 7}", "t", i % 7) for i in range(61)]
    for plan_kw in ({}, dict(record_corruption_rate=0.2, rank_failure_rate=0.3, seed=2)):
        a, ra = ref.run_campaign(lib_ref, ref.SyntheticScorer(), 4, ref.FaultPlan(**plan_kw), ranks_per_job=3,
                                 batch_size=5, retries=2)
        b, rb = harness.run_campaign(lib_own, harness.SyntheticScorer(), 4, harness.FaultPlan(**plan_kw),
                                     ranks_per_job=3, batch_size=5, retries=2)
        assert [tuple(vars(r).values()) for r in a] == [tuple(vars(r).values()) for r in b]
        assert (ra.succeeded, ra.abandoned, ra.attempts, ra.corrupted) == \
            (rb.succeeded, rb.abandoned, rb.attempts, rb.corrupted)


def test_balanced_partitions():
    assert harness.balanced_sizes(10, 3) == [4, 3, 3]
    lib = [harness.PoseRecord("c", "t", i) for i in range(10)]
    jobs = harness.partition(lib, 3, ranks_per_job=2)
    assert [len(j.poses) for j in jobs] == [4, 3, 3]
    assert [len(r) for r in harness.rank_assignments(jobs[0])] == [2, 2]
    with pytest.raises(ValueError):
        harness.partition([], 1)
    with pytest.raises(ValueError):
        harness.partition(lib, 11)


@pytest.mark.gpu
@pytest.mark.parametrize("payload", ["featurized", "raw"])
def test_b200_scorer_behind_campaign_matches_reference(tmp_path, payload):
    """The B200 ModelScorer (fp32 path) behind run_campaign reproduces the
    reference campaign: same records, shards and manifests, scores within
    1e-3 relative.  Payloads: device-featurized (VoxelGrid, ComplexGraph)
    pairs through predict_batch, or raw complexes featurized inside the
    scorer call."""
    from paper_2104_04547_b200 import complexes as cx
    from paper_2104_04547_b200 import models
    z = load("campaign_golden.npz")
    cs = [cx.SyntheticComplex(f"p{i}", pos, el, ro, 0.0) for i, (pos, el, ro) in enumerate(complexes_of(z))]
    vcfg, gcfg = models.VoxelHeadConfig(), models.GraphHeadConfig()
    model = models.FusionModel(vcfg, gcfg, models.table_coherent_fusion_config(), seed=0)
    if payload == "featurized":
        payloads = [(it.grid, it.graph) for it in models.featurize(cs, vcfg, gcfg)]
    else:
        payloads = cs
    out = _run(tmp_path, harness.ModelScorer(model), payloads)
    _check(*out, lambda a, b: np.testing.assert_allclose(a, b, rtol=1e-3))
