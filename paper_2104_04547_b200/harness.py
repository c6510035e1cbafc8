"""Scorer plugin and partitioning helpers of ``fusionscreen.harness`` for the
B200 scoring path (harness.py:37-52, :132-167, :224-234).

``ModelScorer`` keeps the reference plugin contract
``scorer(list[PoseRecord]) -> list[float]`` (used at harness.py:278) and its
error behaviour (``ValueError("unscorable pose <key>: <reason>")``), so
``fusionscreen.harness.run_job``/``run_campaign`` can drive it unchanged.  It
additionally accepts raw ``SyntheticComplex`` payloads, which are featurized
on the GPU inside the same call.  The campaign driver itself
(retries, fault injection, shards, manifests) is orchestration outside the
hot path and is not rebuilt here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .complexes import SyntheticComplex

DEFAULT_RANKS_PER_JOB = 16
DEFAULT_BATCH_SIZE = 56


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


def pose_key(p: PoseRecord) -> str:
    return f"{p.compound_id}/{p.target_id}/{p.pose_id}"


def balanced_sizes(n: int, parts: int) -> list:
    """Contiguous balanced split sizes; any two differ by at most one (:132-137)."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    base, extra = divmod(n, parts)
    return [base + 1 if i < extra else base for i in range(parts)]


def shard_bounds(n: int, parts: int) -> list:
    """[start, stop) of each contiguous balanced shard (rank sharding rule)."""
    out, s = [], 0
    for size in balanced_sizes(n, parts):
        out.append((s, s + size))
        s += size
    return out


def compound_aligned_bounds(compound_of_pose, parts: int) -> list:
    """Contiguous shards that never split a compound's poses: balanced over
    compounds (the owner rule of harness.py:290-297), mapped back to poses."""
    comp = np.asarray(compound_of_pose)
    if len(comp) == 0:
        return [(0, 0)] * parts
    starts = np.flatnonzero(np.r_[True, comp[1:] != comp[:-1]])
    bounds = []
    for a, b in shard_bounds(len(starts), parts):
        s = int(starts[a]) if a < len(starts) else len(comp)
        e = int(starts[b]) if b < len(starts) else len(comp)
        bounds.append((s, e))
    return bounds


class ModelScorer:
    """Scores poses whose payloads are (VoxelGrid, ComplexGraph) pairs, or raw
    SyntheticComplex objects (featurized on device)."""

    def __init__(self, model):
        self.model = model

    def __call__(self, poses: list) -> list:
        payloads = [p.payload for p in poses]
        if payloads and all(isinstance(x, SyntheticComplex) for x in payloads):
            scores, err = self.model.score_complexes(payloads)
            for i, e in enumerate(err):
                if e:
                    raise ValueError(f"unscorable pose {pose_key(poses[i])}: device error flags {int(e)}")
            return [float(s) for s in scores]
        preds, errors = self.model.predict_batch(payloads)
        for idx, reason in errors:
            raise ValueError(f"unscorable pose {pose_key(poses[idx])}: {reason}")
        return [float(p) for p in preds]
