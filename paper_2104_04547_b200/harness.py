"""Scorer plugin and the screening-campaign caller of ``fusionscreen.harness``
for the B200 scoring path (harness.py:37-52, :132-167, :204-434).

``ModelScorer`` keeps the reference plugin contract
``scorer(list[PoseRecord]) -> list[float]`` (called at harness.py:278) and its
error behaviour (``ValueError("unscorable pose <key>: <reason>")``), so the
reference's own ``run_job``/``run_campaign`` can drive it unchanged.  Payloads
are duck-typed: (VoxelGrid, ComplexGraph) pairs -- this package's, the
reference's, or anything with the same attributes -- go through
``predict_batch``; raw complexes (``.positions/.elements/.roles``, e.g. the
reference's ``SyntheticComplex``) are featurized on the GPU inside the same
call.

``run_job``/``run_campaign`` restate the reference's campaign semantics so a
B200 screen keeps them without the reference installed: contiguous balanced
jobs and ranks, deterministic SHA-256 fault draws (corruption is a property
of the pose, failures of the (job, attempt)), exactly-once scoring with
retries, all-or-nothing JSONL shards grouped by compound owner, per-job and
campaign manifests.  Outputs are record-for-record those of the reference
(tests/test_harness_campaign.py replays the reference's goldens).
"""

from __future__ import annotations

import hashlib
import json
import logging
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np

logger = logging.getLogger(__name__)

DEFAULT_RANKS_PER_JOB = 16
DEFAULT_BATCH_SIZE = 56
DEFAULT_LOADERS_PER_RANK = 12
DEFAULT_RETRIES = 3
MANIFEST_NAME = "campaign_manifest.json"


@dataclass(frozen=True)
class PoseRecord:
    compound_id: str
    target_id: str
    pose_id: int
    payload: object = None


@dataclass(frozen=True)
class PredictionRecord:
    compound_id: str
    target_id: str
    pose_id: int
    predicted_pk: float
    job_id: int
    rank_id: int


@dataclass(frozen=True)
class FaultPlan:
    """Deterministic fault injection (harness.py:55-67)."""

    record_corruption_rate: float = 0.0
    rank_failure_rate: float = 0.0
    job_failure_rate: float = 0.0
    seed: int = 0

    def __post_init__(self):
        for name in ("record_corruption_rate", "rank_failure_rate", "job_failure_rate"):
            v = getattr(self, name)
            if not 0.0 <= v < 1.0:
                raise ValueError(f"{name} must be in [0, 1), got {v}")


@dataclass(frozen=True)
class JobSpec:
    job_id: int
    poses: tuple
    ranks_per_job: int = DEFAULT_RANKS_PER_JOB
    batch_size: int = DEFAULT_BATCH_SIZE
    loaders_per_rank: int = DEFAULT_LOADERS_PER_RANK

    def __post_init__(self):
        if min(self.ranks_per_job, self.batch_size, self.loaders_per_rank) < 1:
            raise ValueError("ranks, batch size and loaders must be >= 1")


@dataclass
class JobResult:
    job_id: int
    attempt: int
    status: str
    predictions: list = field(default_factory=list)
    corrupted: list = field(default_factory=list)
    failure_reason: str | None = None
    timings: dict = field(default_factory=dict)


@dataclass
class CampaignReport:
    n_poses: int
    n_jobs: int
    succeeded: list
    abandoned: list
    missing_ranges: list
    attempts: dict
    corrupted: list
    timings: dict

    @property
    def complete(self) -> bool:
        return not self.abandoned


def pose_key(p: PoseRecord) -> str:
    return f"{p.compound_id}/{p.target_id}/{p.pose_id}"


# ---------------------------------------------------------------------------
# partitioning (harness.py:132-167)
# ---------------------------------------------------------------------------

def balanced_sizes(n: int, parts: int) -> list:
    """Contiguous balanced split sizes; any two differ by at most one (:132-137)."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    base, extra = divmod(n, parts)
    return [base + (i < extra) for i in range(parts)]


def shard_bounds(n: int, parts: int) -> list:
    """[start, stop) of each contiguous balanced shard (rank sharding rule)."""
    stops = np.cumsum([0] + balanced_sizes(n, parts))
    return [(int(a), int(b)) for a, b in zip(stops[:-1], stops[1:])]


def compound_aligned_bounds(compound_of_pose, parts: int) -> list:
    """Contiguous shards that never split a compound's poses: balanced over
    compounds (the owner rule of harness.py:290-297), mapped back to poses."""
    comp = np.asarray(compound_of_pose)
    if len(comp) == 0:
        return [(0, 0)] * parts
    starts = np.append(np.flatnonzero(np.r_[True, comp[1:] != comp[:-1]]), len(comp))
    return [(int(starts[a]), int(starts[b])) for a, b in shard_bounds(len(starts) - 1, parts)]


def partition(library: list, n_jobs: int, ranks_per_job: int = DEFAULT_RANKS_PER_JOB,
              batch_size: int = DEFAULT_BATCH_SIZE, loaders_per_rank: int = DEFAULT_LOADERS_PER_RANK) -> list:
    """Contiguous balanced jobs in library order (harness.py:140-158)."""
    if not library:
        raise ValueError("empty library")
    if n_jobs > len(library):
        raise ValueError(f"{n_jobs} jobs for {len(library)} poses")
    return [JobSpec(j, tuple(library[a:b]), ranks_per_job, batch_size, loaders_per_rank)
            for j, (a, b) in enumerate(shard_bounds(len(library), n_jobs))]


def rank_assignments(spec: JobSpec) -> list:
    """Contiguous balanced split of a job's poses over its ranks (:161-167)."""
    return [list(spec.poses[a:b]) for a, b in shard_bounds(len(spec.poses), spec.ranks_per_job)]


# ---------------------------------------------------------------------------
# deterministic fault draws (harness.py:174-197)
# ---------------------------------------------------------------------------

def _unit_hash(*parts) -> float:
    digest = hashlib.sha256(":".join(map(str, parts)).encode()).digest()
    return int.from_bytes(digest[:8], "big") / 2 ** 64


def is_corrupted(pose: PoseRecord, plan: FaultPlan) -> bool:
    return plan.record_corruption_rate > 0.0 and \
        _unit_hash(plan.seed, "corrupt", pose_key(pose)) < plan.record_corruption_rate


def attempt_fails(job_id: int, attempt: int, plan: FaultPlan):
    if _unit_hash(plan.seed, "job", job_id, attempt) < plan.job_failure_rate:
        return "job lost"
    if _unit_hash(plan.seed, "rank", job_id, attempt) < plan.rank_failure_rate:
        return "rank died mid-job"
    return None


# ---------------------------------------------------------------------------
# scorers
# ---------------------------------------------------------------------------

class SyntheticScorer:
    """Hash-based scores in [2, 12) with a sleep cost model (harness.py:204-221);
    the reference's stand-in scorer for harness tests."""

    def __init__(self, per_pose_s: float = 0.0, per_batch_s: float = 0.0, seed: int = 0):
        self.per_pose_s, self.per_batch_s, self.seed = per_pose_s, per_batch_s, seed

    def __call__(self, poses: list) -> list:
        if self.per_pose_s or self.per_batch_s:
            time.sleep(self.per_pose_s * len(poses) + self.per_batch_s)
        return [2.0 + 10.0 * _unit_hash(self.seed, "score", pose_key(p)) for p in poses]


def _is_complex(x) -> bool:
    return all(hasattr(x, a) for a in ("positions", "elements", "roles"))


class ModelScorer:
    """Scores poses whose payloads are (VoxelGrid, ComplexGraph) pairs, or raw
    complexes (featurized on device in the same call)."""

    def __init__(self, model):
        self.model = model

    def __call__(self, poses: list) -> list:
        payloads = [p.payload for p in poses]
        if payloads and all(_is_complex(x) for x in payloads):
            scores, err = self.model.score_complexes(payloads)
            for i, e in enumerate(err):
                if e:
                    raise ValueError(f"unscorable pose {pose_key(poses[i])}: {_device_reason(int(e))}")
            return [float(s) for s in scores]
        preds, errors = self.model.predict_batch(payloads)
        for idx, reason in errors:
            raise ValueError(f"unscorable pose {pose_key(poses[idx])}: {reason}")
        return [float(p) for p in preds]


def _device_reason(e: int) -> str:
    from . import _native as N
    names = [(N.FS_ERR_ROLE, "role outside {PROTEIN, LIGAND}"), (N.FS_ERR_NAN, "non-finite coordinates"),
             (N.FS_ERR_NONFINITE, "non-finite coordinates"), (N.FS_ERR_TOO_LARGE, "too many atoms"),
             (N.FS_ERR_EDGE_CAP, "edge capacity exceeded")]
    why = sorted({s for bit, s in names if e & bit})
    return ", ".join(why) if why else f"device error flags {e}"


# ---------------------------------------------------------------------------
# job and campaign (harness.py:245-424)
# ---------------------------------------------------------------------------

def _write_job_outputs(spec: JobSpec, attempt: int, result: JobResult, out_dir) -> None:
    """Per-rank JSONL shards (each compound owned by one rank, balanced over
    the sorted compound ids) + job manifest + error list (:289-321)."""
    recs = result.predictions
    compounds = sorted({r.compound_id for r in recs})
    owner = {}
    for rank_id, (a, b) in enumerate(shard_bounds(len(compounds), spec.ranks_per_job)):
        owner.update((c, rank_id) for c in compounds[a:b])
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    by_rank = {}
    for r in recs:
        by_rank.setdefault(owner[r.compound_id], []).append(r)
    shard_files = []
    for rank_id in range(spec.ranks_per_job):
        rows = sorted(by_rank.get(rank_id, []), key=lambda r: (r.compound_id, r.target_id, r.pose_id))
        name = f"shard_{spec.job_id:05d}_{rank_id:03d}.jsonl"
        (out_dir / name).write_text("".join(json.dumps(asdict(r)) + "\n" for r in rows))
        shard_files.append({"file": name, "records": len(rows)})
    with open(out_dir / f"job_{spec.job_id:05d}_manifest.json", "w") as f:
        json.dump({"job_id": spec.job_id, "attempt": attempt, "poses": len(spec.poses), "scored": len(recs),
                   "corrupted": len(result.corrupted), "shards": shard_files}, f, indent=2)
    if result.corrupted:
        (out_dir / f"job_{spec.job_id:05d}_errors.jsonl").write_text(
            "".join(json.dumps({"pose": k, "reason": why}) + "\n" for k, why in result.corrupted))


def run_job(spec: JobSpec, scorer, plan: FaultPlan | None = None, attempt: int = 0, out_dir=None) -> JobResult:
    """One job attempt: score every rank's clean poses in batches of
    ``spec.batch_size``, gather, then write shards only if the attempt
    succeeds (harness.py:245-325)."""
    plan = plan or FaultPlan()
    result = JobResult(spec.job_id, attempt, "ok")
    t0 = time.perf_counter()
    ranks = rank_assignments(spec)
    t1 = time.perf_counter()
    reason = attempt_fails(spec.job_id, attempt, plan)
    if reason is not None:
        result.status, result.failure_reason = "failed", reason
        logger.warning("job %d attempt %d failed: %s", spec.job_id, attempt, reason)
        return result
    for rank_id, poses in enumerate(ranks):
        clean = []
        for p in poses:
            if is_corrupted(p, plan):
                result.corrupted.append((pose_key(p), "corrupt record"))
            else:
                clean.append(p)
        for s in range(0, len(clean), spec.batch_size):
            batch = clean[s:s + spec.batch_size]
            result.predictions.extend(PredictionRecord(p.compound_id, p.target_id, p.pose_id, score,
                                                       spec.job_id, rank_id)
                                      for p, score in zip(batch, scorer(batch)))
    t2 = time.perf_counter()
    if out_dir is not None:
        _write_job_outputs(spec, attempt, result, out_dir)
    t3 = time.perf_counter()
    result.timings = {"startup_s": t1 - t0, "evaluation_s": t2 - t1, "output_s": t3 - t2}
    return result


def run_campaign(library: list, scorer, n_jobs: int, plan: FaultPlan | None = None, out_dir=None,
                 parallelism: int = 4, retries: int = DEFAULT_RETRIES, ranks_per_job: int = DEFAULT_RANKS_PER_JOB,
                 batch_size: int = DEFAULT_BATCH_SIZE, loaders_per_rank: int = DEFAULT_LOADERS_PER_RANK):
    """Partition, run jobs on a thread pool, retry failed attempts, report
    abandoned ranges; every pose is scored exactly once (harness.py:348-424).
    Returns (predictions, CampaignReport)."""
    plan = plan or FaultPlan()
    t0 = time.perf_counter()
    jobs = partition(library, n_jobs, ranks_per_job, batch_size, loaders_per_rank)
    attempts = {j.job_id: 0 for j in jobs}
    results, abandoned = {}, []
    pending = list(jobs)
    with ThreadPoolExecutor(max_workers=max(1, parallelism)) as pool:
        while pending:
            futs = [(pool.submit(run_job, j, scorer, plan, attempts[j.job_id], out_dir), j) for j in pending]
            pending = []
            for fut, spec in futs:
                res = fut.result()
                attempts[spec.job_id] += 1
                if res.status == "ok":
                    results[spec.job_id] = res
                elif attempts[spec.job_id] <= retries:
                    pending.append(spec)
                else:
                    abandoned.append(spec.job_id)
                    logger.error("job %d abandoned after %d attempts", spec.job_id, attempts[spec.job_id])
    t1 = time.perf_counter()
    done = [results[j] for j in sorted(results)]
    predictions = [r for res in done for r in res.predictions]
    corrupted = [c for res in done for c in res.corrupted]
    missing = [{"job_id": j, "first": pose_key(jobs[j].poses[0]), "last": pose_key(jobs[j].poses[-1]),
                "count": len(jobs[j].poses)} for j in sorted(abandoned)]
    phase = lambda k: sum(r.timings.get(k, 0.0) for r in done)  # noqa: E731
    report = CampaignReport(n_poses=len(library), n_jobs=n_jobs, succeeded=sorted(results),
                            abandoned=sorted(abandoned), missing_ranges=missing, attempts=attempts,
                            corrupted=corrupted,
                            timings={"wall_s": t1 - t0, "startup_s": phase("startup_s"),
                                     "evaluation_s": phase("evaluation_s"), "output_s": phase("output_s")})
    if out_dir is not None:
        Path(out_dir).mkdir(parents=True, exist_ok=True)
        with open(Path(out_dir) / MANIFEST_NAME, "w") as f:
            json.dump({"n_poses": report.n_poses, "n_jobs": report.n_jobs, "succeeded": report.succeeded,
                       "abandoned": report.abandoned, "missing_ranges": report.missing_ranges,
                       "attempts": attempts, "corrupted": len(corrupted), "complete": report.complete,
                       "timings": report.timings}, f, indent=2)
    return predictions, report


def load_shards(out_dir) -> list:
    """Every shard record of a campaign directory (harness.py:427-434)."""
    out = []
    for path in sorted(Path(out_dir).glob("shard_*.jsonl")):
        with open(path) as f:
            out.extend(PredictionRecord(**json.loads(line)) for line in f)
    return out
