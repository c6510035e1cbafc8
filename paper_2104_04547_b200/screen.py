"""Pocket screening engine: device-resident pose libraries, batched fused
scoring (featurize + 3D-CNN + SG-CNN + fusion in one fs_score_poses call per
batch), running top-k on device, and the multi-GPU merge.

Sharding: each rank owns a contiguous, compound-aligned slice
of the global pose index range and scores it with no data-path collective;
the only exchange is one all-gather of every rank's per-target top-k
(score f32, global pose index i64) over NCCL, merged on every rank with the
same (score desc, index asc) order (tie rule of evaluate.py:67-83).
"""

from __future__ import annotations

import numpy as np
import torch

from . import engine as E
from .synth import Pocket, PoseLibrary


class DeviceLibrary:
    """A PoseLibrary uploaded to one device (positions float64, ids int32)."""

    def __init__(self, lib: PoseLibrary, pockets, device, index_base=0):
        self.lib = lib
        self.device = device
        self.index_base = int(index_base)
        self.xyz = torch.from_numpy(np.ascontiguousarray(lib.xyz)).to(device)
        self.elem = torch.from_numpy(np.ascontiguousarray(lib.elem, dtype=np.int32)).to(device)
        self.role = torch.from_numpy(np.ascontiguousarray(lib.role, dtype=np.int32)).to(device)
        self.atom_off = torch.from_numpy(np.ascontiguousarray(lib.atom_off, dtype=np.int64)).to(device)
        self.target = torch.from_numpy(np.ascontiguousarray(lib.target, dtype=np.int32)).to(device)
        self.pidx = torch.arange(self.index_base, self.index_base + lib.n_poses, dtype=torch.int64, device=device)
        self.compound = torch.from_numpy(np.ascontiguousarray(lib.compound, dtype=np.int64)).to(device)
        self.pose_id = torch.from_numpy(np.ascontiguousarray(lib.pose_id, dtype=np.int64)).to(device)
        p_xyz = np.concatenate([p.xyz for p in pockets])
        p_off = np.concatenate([[0], np.cumsum([len(p.xyz) for p in pockets])]).astype(np.int64)
        self.pocket_xyz = torch.from_numpy(p_xyz).to(device)
        self.pocket_elem = torch.from_numpy(np.concatenate([p.elem for p in pockets]).astype(np.int32)).to(device)
        self.pocket_role = torch.from_numpy(np.concatenate([p.role for p in pockets]).astype(np.int32)).to(device)
        self.pocket_off = torch.from_numpy(p_off).to(device)
        lig = np.diff(lib.atom_off)
        psz = np.diff(p_off)
        self.max_pose_atoms = int((lig + psz[lib.target]).max()) if lib.n_poses else 1

    @property
    def n_poses(self):
        return self.lib.n_poses

    def batch(self, s, e) -> E.PoseBatch:
        return E.PoseBatch(self.xyz, self.elem, self.role, self.atom_off[s:e + 1], self.max_pose_atoms,
                           self.pocket_xyz, self.pocket_elem, self.pocket_role, self.pocket_off,
                           self.target[s:e])

    def batches(self, batch_size):
        """(s, e, PoseBatch, compound, pose_id) per batch; same protocol as
        poselib.StreamingLoader.batches."""
        for s in range(0, self.n_poses, batch_size):
            e = min(self.n_poses, s + batch_size)
            yield s, e, self.batch(s, e), self.compound[s:e], self.pose_id[s:e]


class HostStager:
    """Pinned host copy of a library, pre-cut into batches, for end-to-end
    runs: every step copies its batch's atoms host->device (one
    cudaMemcpyAsync per array) and reads the scores back."""

    def __init__(self, lib: PoseLibrary, batch_size: int, dlib: DeviceLibrary):
        self.lib = lib
        self.B = batch_size
        self.dlib = dlib
        P = lib.n_poses
        self.bounds = [(s, min(P, s + batch_size)) for s in range(0, P, batch_size)]
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        self.h_xyz, self.h_elem, self.h_role = pin(lib.xyz), pin(lib.elem.astype(np.int32)), pin(lib.role.astype(np.int32))
        self.h_target = pin(lib.target.astype(np.int32))
        offs = np.zeros((len(self.bounds), batch_size + 1), dtype=np.int64)
        for i, (s, e) in enumerate(self.bounds):
            offs[i, : e - s + 1] = lib.atom_off[s:e + 1] - lib.atom_off[s]
        self.h_off = pin(offs)
        max_atoms = max(int(lib.atom_off[e] - lib.atom_off[s]) for s, e in self.bounds)
        dev = dlib.device
        self.d_xyz = torch.empty((max_atoms, 3), dtype=torch.float64, device=dev)
        self.d_elem = torch.empty(max_atoms, dtype=torch.int32, device=dev)
        self.d_role = torch.empty(max_atoms, dtype=torch.int32, device=dev)
        self.d_off = torch.empty(batch_size + 1, dtype=torch.int64, device=dev)
        self.d_target = torch.empty(batch_size, dtype=torch.int32, device=dev)
        self.h_scores = torch.empty(batch_size, dtype=torch.float32).pin_memory()

    def stage(self, i):
        """H2D copies of batch i; returns (PoseBatch, h2d bytes)."""
        s, e = self.bounds[i]
        a, b = int(self.lib.atom_off[s]), int(self.lib.atom_off[e])
        n = b - a
        self.d_xyz[:n].copy_(self.h_xyz[a:b], non_blocking=True)
        self.d_elem[:n].copy_(self.h_elem[a:b], non_blocking=True)
        self.d_role[:n].copy_(self.h_role[a:b], non_blocking=True)
        self.d_off[: e - s + 1].copy_(self.h_off[i, : e - s + 1], non_blocking=True)
        self.d_target[: e - s].copy_(self.h_target[s:e], non_blocking=True)
        nbytes = n * (24 + 4 + 4) + (e - s + 1) * 8 + (e - s) * 4
        d = self.dlib
        b_ = E.PoseBatch(self.d_xyz, self.d_elem, self.d_role, self.d_off[: e - s + 1], d.max_pose_atoms,
                         d.pocket_xyz, d.pocket_elem, d.pocket_role, d.pocket_off, self.d_target[: e - s])
        return b_, nbytes

    def read_scores(self, scores):
        n = scores.numel()
        self.h_scores[:n].copy_(scores, non_blocking=True)
        return n * 4


class Screen:
    """Scores a DeviceLibrary batch by batch with a running device top-k.

    ``pocket_cache`` (DeviceModel.prepare_pockets of the library's pockets)
    switches to the pocket-factored scorer: same
    scores to fp32 rounding; non-factorable poses come back flagged
    FS_ERR_NOT_FACTORED (rescore them with a plain Screen)."""

    def __init__(self, model: E.DeviceModel, precision="bf16", batch_size=8192, k=100,
                 max_edges_per_pose=32768, pocket_cache=None):
        if pocket_cache is not None and precision != pocket_cache.precision:
            raise ValueError(f"pocket cache prepared at {pocket_cache.precision!r}, screen runs {precision!r}")
        self.model = model
        self.precision = precision
        self.B = batch_size
        self.k = k
        self.max_edges_per_pose = max_edges_per_pose
        self.pocket_cache = pocket_cache

    def score(self, batch: E.PoseBatch, outputs=("scores",)):
        # no host sync: overflow shows up in err (checked after the screen)
        if self.pocket_cache is not None:
            return self.model.score_poses_cached(batch, self.pocket_cache, self.max_edges_per_pose, outputs,
                                                 rescore=False)
        return self.model.score_poses(batch, self.precision, self.max_edges_per_pose, outputs, retry=False)

    def run(self, source, keep_scores=False, best_compounds=None, compound_base=0, direction="max"):
        """Score a whole library -- a DeviceLibrary (resident in HBM) or a
        poselib.StreamingLoader (pinned host streaming).  Returns
        dict(topk_scores, topk_idx, err, scores?): the running top-k over
        poses, pose indices global (source.index_base + local).

        With ``best_compounds=C`` the per-compound best pose (rule of
        evaluate.aggregate_best_pose, evaluate.py:67-83) is folded batch by
        batch on device for compounds [compound_base, compound_base + C)
        and the result adds best_score[C], best_pose[C] and the top-k over
        compounds (topk_compound_scores, topk_compound_idx)."""
        top_s = top_i = None
        errs, all_s = [], []
        acc = (E.BestPoseAccumulator(best_compounds, compound_base, direction)
               if best_compounds is not None else None)
        base = source.index_base
        for s, e, batch, compound, pose_id in source.batches(self.B):
            out = self.score(batch)
            pidx = torch.arange(base + s, base + e, dtype=torch.int64, device=out["scores"].device)
            top_s, top_i = E.topk_merge(top_s, top_i, out["scores"], pidx, self.k)
            if acc is not None:
                acc.update(compound, pose_id, out["scores"])
            errs.append(out["err"])
            if keep_scores:
                all_s.append(out["scores"])
        res = {"topk_scores": top_s, "topk_idx": top_i, "err": torch.cat(errs) if errs else None}
        if keep_scores:
            res["scores"] = torch.cat(all_s)
        if acc is not None:
            res.update(compound_topk(acc, self.k))
        return res


def compound_topk(acc: E.BestPoseAccumulator, k):
    """Decode a best-pose accumulator and rank its compounds: dict(best_score,
    best_pose, topk_compound_scores, topk_compound_idx); compound ids are
    global (acc.base + local), ties to the lower id, compounds without a
    scored pose last."""
    bs, bp = acc.result()
    cid = torch.arange(acc.base, acc.base + acc.n, dtype=torch.int64, device=bs.device)
    ranked = bs if acc.dir > 0 else -bs
    cs, ci = E.topk_merge(None, None, ranked, cid, k)
    return {"best_score": bs, "best_pose": bp, "topk_compound_scores": cs if acc.dir > 0 else -cs,
            "topk_compound_idx": ci}


def merge_topk_across_ranks(top_s, top_i, k, group=None, merge=None, device=None):
    """All-gather every rank's top-k (NCCL over NVLink) and merge on device.
    Ranks holding fewer than k entries -- or none (an empty shard: ``top_s``
    None) -- pad with NaN scores (ranked last) and the largest index, so every
    rank joins the collective.  `merge` defaults to the device kernel
    fs_topk_merge (tests pass a CPU rule)."""
    import torch.distributed as dist
    merge = merge or (lambda s, i, kk: E.topk_merge(s, i, None, None, kk))
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return top_s, top_i
    if device is None:
        device = top_s.device if top_s is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
    ws = dist.get_world_size(group)
    pad_s = torch.full((k,), float("nan"), dtype=torch.float32, device=device)
    pad_i = torch.full((k,), np.iinfo(np.int64).max, dtype=torch.int64, device=device)
    if top_s is not None and top_s.numel():
        pad_s[: top_s.numel()] = top_s
        pad_i[: top_i.numel()] = top_i
    gs = torch.empty(ws * k, dtype=torch.float32, device=device)
    gi = torch.empty(ws * k, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(gs, pad_s, group=group)
    dist.all_gather_into_tensor(gi, pad_i, group=group)
    # fewer than k entries over all ranks leave trailing pads (NaN, int64 max)
    return merge(gs, gi, k)
