"""Device-side engine: pose batches, packed models, workspaces, and the calls
through the C-ABI.  Torch provides device memory and the current stream only.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N


def _require_cuda(device=None):
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2104_04547_b200 needs a CUDA device (B200); there is no CPU path")
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


# ---------------------------------------------------------------------------
# pose batches
# ---------------------------------------------------------------------------

@dataclass
class PoseBatch:
    """Device-resident batch of poses (see fs_pose_batch in include/fusionb200.h).

    Pose p = pocket atoms of ``pose_target[p]`` (if any) followed by its own
    atoms, i.e. the reference's ``np.vstack([prot, lig])`` node order
    (complexes.py:114-118).
    """

    atom_xyz: torch.Tensor          # [A,3] float64
    atom_elem: torch.Tensor         # [A] int32
    atom_role: torch.Tensor         # [A] int32
    atom_off: torch.Tensor          # [P+1] int64
    max_pose_atoms: int
    pocket_xyz: torch.Tensor | None = None
    pocket_elem: torch.Tensor | None = None
    pocket_role: torch.Tensor | None = None
    pocket_off: torch.Tensor | None = None
    pose_target: torch.Tensor | None = None
    n_nodes: int | None = None      # host-known total node count (optional)

    @property
    def n_poses(self) -> int:
        return int(self.atom_off.numel()) - 1

    @property
    def device(self):
        return self.atom_xyz.device

    def cstruct(self) -> N.PoseBatchC:
        s = N.PoseBatchC()
        s.pocket_xyz = self.pocket_xyz.data_ptr() if self.pocket_xyz is not None else None
        s.pocket_elem = self.pocket_elem.data_ptr() if self.pocket_elem is not None else None
        s.pocket_role = self.pocket_role.data_ptr() if self.pocket_role is not None else None
        s.pocket_off = self.pocket_off.data_ptr() if self.pocket_off is not None else None
        s.n_pockets = 0 if self.pocket_off is None else int(self.pocket_off.numel()) - 1
        s.atom_xyz = self.atom_xyz.data_ptr()
        s.atom_elem = self.atom_elem.data_ptr()
        s.atom_role = self.atom_role.data_ptr()
        s.atom_off = self.atom_off.data_ptr()
        s.pose_target = self.pose_target.data_ptr() if self.pose_target is not None else None
        s.n_poses = self.n_poses
        s.max_pose_atoms = int(self.max_pose_atoms)
        return s

    def slice(self, start: int, stop: int) -> "PoseBatch":
        """Poses [start, stop) as a view (offsets rebased on device)."""
        off = self.atom_off[start:stop + 1]
        return PoseBatch(self.atom_xyz, self.atom_elem, self.atom_role, off, self.max_pose_atoms,
                         self.pocket_xyz, self.pocket_elem, self.pocket_role, self.pocket_off,
                         None if self.pose_target is None else self.pose_target[start:stop])


def _int32_checked(a, what):
    a = np.asarray(a)
    if a.size and (a.min() < np.iinfo(np.int32).min or a.max() > np.iinfo(np.int32).max):
        # clip keeps the reference semantics for elements (clipped to c_elem-1);
        # an out-of-range role stays invalid after clipping.
        a = np.clip(a, np.iinfo(np.int32).min, np.iinfo(np.int32).max)
    return np.ascontiguousarray(a, dtype=np.int32)


def batch_from_arrays(positions, elements, roles, atom_off, device=None,
                      pocket=None, pose_target=None) -> PoseBatch:
    """Upload host arrays (float64 positions, integer elements/roles)."""
    dev = _require_cuda(device)
    atom_off = np.ascontiguousarray(atom_off, dtype=np.int64)
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    counts = np.diff(atom_off)
    kw = {}
    pocket_counts = np.zeros(len(counts), dtype=np.int64)
    if pocket is not None:
        ppos, pel, pro, poff = pocket
        poff = np.ascontiguousarray(poff, dtype=np.int64)
        kw = dict(pocket_xyz=torch.from_numpy(np.ascontiguousarray(ppos, dtype=np.float64).reshape(-1, 3)).to(dev),
                  pocket_elem=torch.from_numpy(_int32_checked(pel, "elem")).to(dev),
                  pocket_role=torch.from_numpy(_int32_checked(pro, "role")).to(dev),
                  pocket_off=torch.from_numpy(poff).to(dev))
        tgt = np.ascontiguousarray(pose_target, dtype=np.int32)
        kw["pose_target"] = torch.from_numpy(tgt).to(dev)
        psz = np.diff(poff)
        pocket_counts = np.where(tgt >= 0, psz[np.maximum(tgt, 0)], 0)
    nodes = counts + pocket_counts
    maxn = int(nodes.max()) if len(nodes) else 1
    return PoseBatch(atom_xyz=torch.from_numpy(pos).to(dev),
                     atom_elem=torch.from_numpy(_int32_checked(elements, "elem")).to(dev),
                     atom_role=torch.from_numpy(_int32_checked(roles, "role")).to(dev),
                     atom_off=torch.from_numpy(atom_off).to(dev),
                     max_pose_atoms=max(maxn, 1), n_nodes=int(nodes.sum()), **kw)


_STAGE = threading.local()


def _pinned(name, numel, dtype):
    """Per-thread pinned host staging buffer (grown on demand)."""
    buf = getattr(_STAGE, name, None)
    if buf is None or buf.numel() < numel:
        buf = torch.empty(max(int(numel * 1.25), 1024), dtype=dtype).pin_memory()
        setattr(_STAGE, name, buf)
    return buf


def batch_from_complexes(complexes, device=None) -> PoseBatch:
    """SyntheticComplex-like objects (positions/elements/roles) -> PoseBatch.

    Each complex is copied once, straight into per-thread pinned staging
    buffers (float64 xyz; elements and roles as int64, a plain copy of the
    reference's integer arrays), uploaded with one asynchronous DMA per
    array, and narrowed to int32 on the device with values clipped to the
    int32 range (which keeps the reference's element clipping and leaves an
    invalid role invalid).  The staging buffers are reused by the thread's
    next call, which the caller orders after this batch's scores are read
    back."""
    dev = _require_cuda(device)
    counts = np.fromiter((len(c.positions) for c in complexes), dtype=np.int64, count=len(complexes))
    off = np.zeros(len(complexes) + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    A = int(off[-1])
    h_xyz = _pinned("xyz", 3 * A, torch.float64)[: 3 * A]
    h_el = _pinned("elem", A, torch.int64)[:A]
    h_ro = _pinned("role", A, torch.int64)[:A]
    x, e_, r_ = h_xyz.numpy().reshape(-1, 3), h_el.numpy(), h_ro.numpy()
    for c, a, b in zip(complexes, off[:-1], off[1:]):
        x[a:b] = c.positions
        e_[a:b] = c.elements
        r_[a:b] = c.roles
    lo, hi = np.iinfo(np.int32).min, np.iinfo(np.int32).max
    d_el = h_el.to(dev, non_blocking=True).clamp_(lo, hi).to(torch.int32)
    d_ro = h_ro.to(dev, non_blocking=True).clamp_(lo, hi).to(torch.int32)
    maxn = int(counts.max()) if len(counts) else 1
    return PoseBatch(atom_xyz=h_xyz.to(dev, non_blocking=True).view(-1, 3), atom_elem=d_el, atom_role=d_ro,
                     atom_off=torch.from_numpy(off).to(dev), max_pose_atoms=max(maxn, 1), n_nodes=A)


def node_offsets(batch: PoseBatch) -> torch.Tensor:
    L = N.lib()
    node_off = torch.empty(batch.n_poses + 1, dtype=torch.int64, device=batch.device)
    ws = torch.empty(L.fs_node_offsets_ws_bytes(batch.n_poses), dtype=torch.uint8, device=batch.device)
    s = batch.cstruct()
    N.check(L.fs_node_offsets(C.byref(s), _ptr(node_off), _ptr(ws), ws.numel(), _stream()),
            "fs_node_offsets")
    return node_off


# ---------------------------------------------------------------------------
# featurizer calls
# ---------------------------------------------------------------------------

def voxelize(batch: PoseBatch, extent=16, c_elem=4, box_size=16.0, layout=N.FS_GRID_NCDHW_F64):
    """complexes.voxelize (complexes.py:171-184) for a whole batch on device."""
    if extent < 8:
        raise ValueError(f"grid extent must be >= 8, got {extent}")
    L = N.lib()
    P, ch = batch.n_poses, 2 * c_elem
    if layout == N.FS_GRID_NCDHW_F64:
        out = torch.empty((P, ch, extent, extent, extent), dtype=torch.float64, device=batch.device)
    elif layout == N.FS_GRID_NDHWC_F32:
        out = torch.empty((P, extent, extent, extent, ch), dtype=torch.float32, device=batch.device)
    else:
        out = torch.empty((P, extent, extent, extent, ch), dtype=torch.bfloat16, device=batch.device)
    err = torch.zeros(P, dtype=torch.int32, device=batch.device)
    s = batch.cstruct()
    N.check(L.fs_voxelize(C.byref(s), extent, c_elem, float(box_size), layout, _ptr(out), _ptr(err),
                          _stream()), "fs_voxelize")
    return out, err


@dataclass
class DeviceGraph:
    node_off: torch.Tensor
    row_cov: torch.Tensor
    col_cov: torch.Tensor
    dist_cov: torch.Tensor | None
    row_ncov: torch.Tensor
    col_ncov: torch.Tensor
    dist_ncov: torch.Tensor | None
    err: torch.Tensor


def radius_graph(batch: PoseBatch, cov_thresh=2.24, noncov_thresh=5.22, with_dists=True) -> DeviceGraph:
    """Exact covalent / non-covalent CSR per pose (complexes.py:237-246)."""
    lo, hi = 1.2, 5.9
    for t in (cov_thresh, noncov_thresh):
        if not lo <= t <= hi:
            raise ValueError(f"threshold {t} outside searched range [{lo}, {hi}]")
    L = N.lib()
    dev = batch.device
    node_off = node_offsets(batch)
    n = int(node_off[-1].item())
    err = torch.zeros(batch.n_poses, dtype=torch.int32, device=dev)
    dc = torch.empty(n, dtype=torch.int32, device=dev)
    dn = torch.empty(n, dtype=torch.int32, device=dev)
    s = batch.cstruct()
    N.check(L.fs_graph_count(C.byref(s), _ptr(node_off), cov_thresh, noncov_thresh, _ptr(dc), _ptr(dn),
                             _ptr(err), _stream()), "fs_graph_count")
    ws = torch.empty(L.fs_graph_rows_ws_bytes(n), dtype=torch.uint8, device=dev)
    rc_ = torch.empty(n + 1, dtype=torch.int64, device=dev)
    rn_ = torch.empty(n + 1, dtype=torch.int64, device=dev)
    N.check(L.fs_graph_rows(_ptr(dc), n, _ptr(rc_), _ptr(ws), ws.numel(), _stream()), "fs_graph_rows")
    N.check(L.fs_graph_rows(_ptr(dn), n, _ptr(rn_), _ptr(ws), ws.numel(), _stream()), "fs_graph_rows")
    ec, en = int(rc_[-1].item()), int(rn_[-1].item())
    col_c = torch.empty(max(ec, 1), dtype=torch.int32, device=dev)
    col_n = torch.empty(max(en, 1), dtype=torch.int32, device=dev)
    d_c = torch.empty(max(ec, 1), dtype=torch.float64, device=dev) if with_dists else None
    d_n = torch.empty(max(en, 1), dtype=torch.float64, device=dev) if with_dists else None
    N.check(L.fs_graph_fill(C.byref(s), _ptr(node_off), cov_thresh, noncov_thresh, _ptr(rc_), _ptr(rn_),
                            _ptr(col_c), _ptr(col_n), _ptr(d_c), _ptr(d_n), ec, en, _ptr(err), _stream()),
            "fs_graph_fill")
    return DeviceGraph(node_off, rc_, col_c[:ec], None if d_c is None else d_c[:ec], rn_, col_n[:en],
                       None if d_n is None else d_n[:en], err)


def edge_lists(g: DeviceGraph, which="cov"):
    """i<j pairs (pose-local ids) of one edge type, lexsorted, per pose offsets."""
    L = N.lib()
    dev = g.node_off.device
    P = g.node_off.numel() - 1
    row, col, dist = (g.row_cov, g.col_cov, g.dist_cov) if which == "cov" else (g.row_ncov, g.col_ncov, g.dist_ncov)
    edge_off = torch.empty(P + 1, dtype=torch.int64, device=dev)
    ws = torch.empty(L.fs_node_offsets_ws_bytes(P) + 1024, dtype=torch.uint8, device=dev)
    colp = col if col.numel() else torch.empty(1, dtype=torch.int32, device=dev)
    N.check(L.fs_graph_edge_counts(_ptr(g.node_off), P, _ptr(row), _ptr(colp), _ptr(edge_off), _ptr(ws),
                                   ws.numel(), _stream()), "fs_graph_edge_counts")
    e = int(edge_off[-1].item())
    edges = torch.empty((max(e, 1), 2), dtype=torch.int64, device=dev)
    dists = torch.empty(max(e, 1), dtype=torch.float64, device=dev) if dist is not None else None
    N.check(L.fs_graph_edges(_ptr(g.node_off), P, _ptr(row), _ptr(colp), _ptr(dist), _ptr(edge_off),
                             _ptr(edges), _ptr(dists), _stream()), "fs_graph_edges")
    return edges[:e], (None if dists is None else dists[:e]), edge_off


def scoring_graph_entries(batch: PoseBatch, cov_thresh=2.24, noncov_thresh=5.22, max_edges=32768,
                          factored=False, max_pocket_atoms=0, c_elem=4, box_size=16.0, with_dists=True):
    """The radius graph exactly as the scoring path builds it (fs_scoring_graph):
    dict(n_cov [P], n_ncov [P], ent_cov [P, max_edges, 2], ent_ncov, d_cov
    [P, max_edges], d_ncov, err [P]) -- directed CSR entries per pose in the
    pose's original node numbering; only the first n_*[p] of each are set."""
    L = N.lib()
    dev = batch.device
    P = batch.n_poses
    nbytes = L.fs_scoring_graph_ws_bytes(P, batch.max_pose_atoms, max_edges, int(bool(factored)), c_elem)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    out = {"n_cov": torch.zeros(P, dtype=torch.int32, device=dev),
           "n_ncov": torch.zeros(P, dtype=torch.int32, device=dev),
           "ent_cov": torch.empty((P, max_edges, 2), dtype=torch.int32, device=dev),
           "ent_ncov": torch.empty((P, max_edges, 2), dtype=torch.int32, device=dev),
           "err": torch.empty(P, dtype=torch.int32, device=dev)}
    if with_dists:
        out["d_cov"] = torch.empty((P, max_edges), dtype=torch.float64, device=dev)
        out["d_ncov"] = torch.empty((P, max_edges), dtype=torch.float64, device=dev)
    s = batch.cstruct()
    N.check(L.fs_scoring_graph(C.byref(s), cov_thresh, noncov_thresh, max_edges, int(bool(factored)),
                               int(max_pocket_atoms), c_elem, float(box_size), _ptr(ws), ws.numel(),
                               _ptr(out["n_cov"]), _ptr(out["n_ncov"]), _ptr(out["ent_cov"]), _ptr(out["ent_ncov"]),
                               _ptr(out.get("d_cov")), _ptr(out.get("d_ncov")), _ptr(out["err"]), _stream()),
            "fs_scoring_graph")
    return out


def node_features(batch: PoseBatch, node_off, c_elem=4, box_size=16.0):
    L = N.lib()
    n = int(node_off[-1].item())
    out = torch.empty((n, c_elem + 4), dtype=torch.float64, device=batch.device)
    s = batch.cstruct()
    N.check(L.fs_node_features(C.byref(s), _ptr(node_off), c_elem, float(box_size), _ptr(out), _stream()),
            "fs_node_features")
    return out


# ---------------------------------------------------------------------------
# packed model
# ---------------------------------------------------------------------------

_ACT = {"relu": 0, "leaky-relu": 1, "selu": 2}
_MODE = {"late": N.FS_MODE_LATE, "mid": N.FS_MODE_MID, "coherent": N.FS_MODE_COHERENT}


def _g(cfg, name):
    return cfg[name] if isinstance(cfg, dict) else getattr(cfg, name)


def model_desc(vcfg, gcfg, fcfg, box_size=16.0) -> N.ModelDescC:
    d = N.ModelDescC()
    for f in ("grid_extent", "in_channels", "conv_filters_1", "conv_filters_2", "dense_nodes",
              "kernel_1", "kernel_2"):
        setattr(d, f, int(_g(vcfg, f)))
    for f in ("residual_1", "residual_2", "batch_norm"):
        setattr(d, f, int(bool(_g(vcfg, f))))
    for f in ("c_elem", "k_cov", "k_noncov", "gather_width_cov", "gather_width_noncov"):
        setattr(d, f, int(_g(gcfg, f)))
    d.cov_thresh = float(_g(gcfg, "cov_thresh"))
    d.noncov_thresh = float(_g(gcfg, "noncov_thresh"))
    d.box_size = float(box_size)
    d.fusion_mode = _MODE[_g(fcfg, "mode")]
    d.n_fusion_layers = int(_g(fcfg, "n_fusion_layers"))
    d.model_specific_layers = int(bool(_g(fcfg, "model_specific_layers")))
    d.residual_fusion = int(bool(_g(fcfg, "residual_fusion")))
    d.activation = _ACT[_g(fcfg, "activation")]
    d.fusion_dense_nodes = int(_g(fcfg, "fusion_dense_nodes"))
    return d


class DeviceModel:
    """Immutable packed weights on one device (fs_model_create)."""

    def __init__(self, vcfg, gcfg, fcfg, flat_params: dict, box_size=16.0, device=None,
                 bn_state: dict | None = None):
        self.device = _require_cuda(device)
        self.vcfg, self.gcfg, self.fcfg = vcfg, gcfg, fcfg
        self.box_size = float(box_size)
        L = N.lib()
        self.desc = model_desc(vcfg, gcfg, fcfg, box_size)
        nbytes = L.fs_weights_bytes(C.byref(self.desc))
        if nbytes == 0:
            raise ValueError("model configuration rejected by fs_weights_bytes")
        params = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in flat_params.items()}
        for key, st in (bn_state or {}).items():          # "bn1" -> {"mean","var"}
            params[f"voxel/{key}_mean"] = np.ascontiguousarray(st["mean"], dtype=np.float64)
            params[f"voxel/{key}_var"] = np.ascontiguousarray(st["var"], dtype=np.float64)
        names = list(params)
        c_names = (C.c_char_p * len(names))(*[n.encode() for n in names])
        c_ptrs = (C.c_void_p * len(names))(*[params[n].ctypes.data for n in names])
        self._keep = params
        with torch.cuda.device(self.device):
            self.blob = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            handle = C.c_void_p()
            N.check(L.fs_model_create(C.byref(self.desc), c_names, c_ptrs, len(names), _ptr(self.blob),
                                      nbytes, _stream(), C.byref(handle)), "fs_model_create")
        self.handle = handle
        # workspaces are per host thread: the reference runs scorer plugins
        # concurrently from a thread pool (harness.py:374-376) and a frozen
        # model must be safe for concurrent prediction; the
        # packed weight blob is read-only
        self._tls = threading.local()

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                N.lib().fs_model_destroy(self.handle)
        except Exception:
            pass

    def supports(self, precision: str) -> bool:
        return bool(N.lib().fs_model_supports(self.handle, N.PRECISIONS[precision]))

    @property
    def latent_v(self):
        return int(_g(self.vcfg, "dense_nodes")) // 2

    @property
    def latent_g(self):
        return int(_g(self.gcfg, "gather_width_noncov"))

    def workspace(self, nbytes: int) -> torch.Tensor:
        ws = getattr(self._tls, "ws", None)
        if ws is None or ws.numel() < nbytes:
            self._tls.ws = None
            ws = torch.empty(int(nbytes * 1.25) + 4096, dtype=torch.uint8, device=self.device)
            self._tls.ws = ws
        return ws

    # -- scoring --------------------------------------------------------------
    def score_poses(self, batch: PoseBatch, precision="fp32", max_edges_per_pose=40000,
                    outputs=("scores",), retry=True, sync_errors=True):
        """featurize + both heads + fusion on device; returns dict of tensors.

        If any pose overflowed the CSR workspace (FS_ERR_EDGE_CAP) the batch is
        re-run with a larger capacity (needs a host read of err when retry)."""
        L = N.lib()
        prec = N.PRECISIONS[precision]
        P = batch.n_poses
        dev = self.device
        out = {"scores": torch.empty(P, dtype=torch.float32, device=dev),
               "err": torch.empty(P, dtype=torch.int32, device=dev)}
        if "lat_v" in outputs:
            out["lat_v"] = torch.empty((P, self.latent_v), dtype=torch.float32, device=dev)
        if "lat_g" in outputs:
            out["lat_g"] = torch.empty((P, self.latent_g), dtype=torch.float32, device=dev)
        if "pred_v" in outputs:
            out["pred_v"] = torch.empty(P, dtype=torch.float32, device=dev)
        if "pred_g" in outputs:
            out["pred_g"] = torch.empty(P, dtype=torch.float32, device=dev)
        cap = int(max_edges_per_pose)
        s = batch.cstruct()
        while True:
            nbytes = L.fs_workspace_bytes(self.handle, P, P * batch.max_pose_atoms, max(1, P) * cap, prec)
            ws = self.workspace(nbytes)
            N.check(L.fs_score_poses(self.handle, prec, C.byref(s), cap, _ptr(ws), ws.numel(),
                                     _ptr(out["scores"]), _ptr(out.get("lat_v")), _ptr(out.get("lat_g")),
                                     _ptr(out.get("pred_v")), _ptr(out.get("pred_g")), _ptr(out["err"]),
                                     _stream()), "fs_score_poses")
            if not retry:
                return out
            if not sync_errors or not bool(((out["err"] & N.FS_ERR_EDGE_CAP) != 0).any().item()):
                return out
            cap *= 2

    # ---- pocket-invariant factoring ----
    def prepare_pockets(self, pocket_xyz, pocket_elem, pocket_role, pocket_off, precision="bf16"):
        """Build the pocket cache (fs_pocket_prepare) for the given device
        pocket arrays (fs_pose_batch layout) at `precision` ("bf16" or
        "mixed"; the cache scores only at that precision).  Returns a
        PocketCache."""
        if precision not in ("bf16", "mixed"):
            raise ValueError(f"pocket factoring runs at bf16 or mixed precision, not {precision!r}")
        L = N.lib()
        off_h = pocket_off.cpu().numpy()
        n = len(off_h) - 1
        mp = int(np.diff(off_h).max()) if n else 1
        stride = L.fs_pocket_cache_bytes(self.handle, mp)
        if stride == 0:
            raise RuntimeError("pocket factoring is not supported for this model / pocket size")
        cache = torch.empty(max(n, 1) * stride, dtype=torch.uint8, device=self.device)
        err = torch.zeros(max(n, 1), dtype=torch.int32, device=self.device)
        ws = self.workspace(L.fs_pocket_prepare_ws_bytes(self.handle, n, mp))
        N.check(L.fs_pocket_prepare(self.handle, N.PRECISIONS[precision], _ptr(pocket_xyz), _ptr(pocket_elem), _ptr(pocket_role),
                                    _ptr(pocket_off), n, mp, _ptr(cache), _ptr(err), _ptr(ws), ws.numel(),
                                    _stream()), "fs_pocket_prepare")
        bad = err[:n].cpu().numpy()
        if bad.any():
            raise ValueError(f"pocket preparation failed (err bits {bad.tolist()})")
        return PocketCache(cache, err, n, mp, stride, precision)

    def score_poses_cached(self, batch: PoseBatch, cache: "PocketCache", max_edges_per_pose=32768,
                           outputs=("scores",), rescore=True):
        """fs_score_poses_cached at the cache's precision: scores from ligand
        atoms + the pocket cache.  Poses flagged FS_ERR_NOT_FACTORED (or
        EDGE_CAP) are re-scored through the full path when `rescore` (needs a
        host read of err)."""
        L = N.lib()
        prec = N.PRECISIONS[cache.precision]
        P = batch.n_poses
        dev = self.device
        out = {"scores": torch.empty(P, dtype=torch.float32, device=dev),
               "err": torch.empty(P, dtype=torch.int32, device=dev)}
        for k, shape in (("lat_v", (P, self.latent_v)), ("lat_g", (P, self.latent_g)), ("pred_v", (P,)),
                         ("pred_g", (P,))):
            if k in outputs:
                out[k] = torch.empty(shape, dtype=torch.float32, device=dev)
        cap = int(max_edges_per_pose)
        S = (batch.max_pose_atoms + 15) // 16 * 16 + 32
        nbytes = L.fs_workspace_bytes(self.handle, P, P * S, max(1, P) * cap, prec)
        ws = self.workspace(nbytes)
        s = batch.cstruct()
        N.check(L.fs_score_poses_cached(self.handle, prec, C.byref(s), _ptr(cache.buf),
                                        cache.max_pocket_atoms, cap, _ptr(ws), ws.numel(), _ptr(out["scores"]),
                                        _ptr(out.get("lat_v")), _ptr(out.get("lat_g")), _ptr(out.get("pred_v")),
                                        _ptr(out.get("pred_g")), _ptr(out["err"]), _stream()),
                "fs_score_poses_cached")
        if rescore:
            redo = ((out["err"] & (N.FS_ERR_NOT_FACTORED | N.FS_ERR_EDGE_CAP)) != 0).nonzero().flatten()
            if redo.numel():
                full = self.score_poses(batch, cache.precision, max_edges_per_pose, outputs)
                for k, v in out.items():
                    v[redo] = full[k][redo]
        return out

    def score_features(self, n_poses, grids=None, feats=None, node_off=None, cov_edges=None,
                       ncov_edges=None, heads=7, precision="fp32", max_pose_nodes=None):
        """Pre-featurized batch (drop-in predict_batch / head forwards).
        ``max_pose_nodes``: the largest pose's node count (read from node_off
        when not given)."""
        if max_pose_nodes is None:
            max_pose_nodes = int((node_off[1:] - node_off[:-1]).max().item()) if node_off is not None and \
                node_off.numel() > 1 else 0
        L = N.lib()
        prec = N.PRECISIONS[precision]
        dev = self.device
        P = int(n_poses)
        n_nodes = 0 if feats is None else int(feats.shape[0])
        ce = cov_edges if cov_edges is not None else torch.empty((0, 2), dtype=torch.int64, device=dev)
        ne = ncov_edges if ncov_edges is not None else torch.empty((0, 2), dtype=torch.int64, device=dev)
        nc, nn = int(ce.shape[0]), int(ne.shape[0])
        nbytes = L.fs_features_workspace_bytes(self.handle, P, n_nodes, int(max_pose_nodes), max(nc, nn), prec)
        ws = self.workspace(nbytes)
        out = {"err": torch.empty(P, dtype=torch.int32, device=dev),
               "scores": torch.empty(P, dtype=torch.float32, device=dev),
               "lat_v": torch.empty((P, self.latent_v), dtype=torch.float32, device=dev),
               "lat_g": torch.empty((P, self.latent_g), dtype=torch.float32, device=dev),
               "pred_v": torch.empty(P, dtype=torch.float32, device=dev),
               "pred_g": torch.empty(P, dtype=torch.float32, device=dev)}
        ce_p = ce if nc else torch.empty(2, dtype=torch.int64, device=dev)
        ne_p = ne if nn else torch.empty(2, dtype=torch.int64, device=dev)
        N.check(L.fs_score_features(self.handle, prec, P, _ptr(grids), _ptr(feats), _ptr(node_off), n_nodes,
                                    int(max_pose_nodes),
                                    _ptr(ce_p), nc, _ptr(ne_p), nn, heads, _ptr(ws), ws.numel(),
                                    _ptr(out["scores"]), _ptr(out["lat_v"]), _ptr(out["lat_g"]),
                                    _ptr(out["pred_v"]), _ptr(out["pred_g"]), _ptr(out["err"]), _stream()),
                "fs_score_features")
        return out


# ---------------------------------------------------------------------------
# ranking
# ---------------------------------------------------------------------------

def topk_merge(a_scores, a_idx, b_scores, b_idx, k):
    """Top-k of the union by (score desc, index asc); NaN last."""
    L = N.lib()
    dev = (a_scores if a_scores is not None else b_scores).device
    na = 0 if a_scores is None else a_scores.numel()
    nb = 0 if b_scores is None else b_scores.numel()
    kk = min(k, na + nb)
    out_s = torch.empty(max(kk, 1), dtype=torch.float32, device=dev)
    out_i = torch.empty(max(kk, 1), dtype=torch.int64, device=dev)
    ws = torch.empty(L.fs_topk_ws_bytes(na + nb) + 1024, dtype=torch.uint8, device=dev)
    N.check(L.fs_topk_merge(_ptr(a_scores), _ptr(a_idx), na, _ptr(b_scores), _ptr(b_idx), nb, kk,
                            _ptr(out_s), _ptr(out_i), _ptr(ws), ws.numel(), _stream()), "fs_topk_merge")
    return out_s[:kk], out_i[:kk]


def best_pose(compound, pose_id, scores, n_compounds, direction="max"):
    if direction not in ("max", "min"):
        raise ValueError(f"direction must be max or min, got {direction!r}")
    L = N.lib()
    dev = scores.device
    idx = torch.empty(max(n_compounds, 1), dtype=torch.int64, device=dev)
    key = torch.empty(max(n_compounds, 1), dtype=torch.int64, device=dev)
    N.check(L.fs_best_pose(_ptr(compound), _ptr(pose_id), _ptr(scores), scores.numel(), n_compounds,
                           1 if direction == "max" else -1, _ptr(idx), _ptr(key), _stream()), "fs_best_pose")
    return idx[:n_compounds]


@dataclass
class PocketCache:
    """Device pocket cache of fs_pocket_prepare (one slot of `stride` bytes per
    pocket, in the order of the pocket arrays it was prepared from)."""

    buf: torch.Tensor
    err: torch.Tensor
    n_pockets: int
    max_pocket_atoms: int
    stride: int
    precision: str = "bf16"


class BestPoseAccumulator:
    """Per-compound best pose folded batch by batch on device
    (fs_best_pose_update/decode; rule of evaluate.aggregate_best_pose)."""

    def __init__(self, n_compounds, compound_base=0, direction="max", device=None):
        if direction not in ("max", "min"):
            raise ValueError(f"direction must be max or min, got {direction!r}")
        self.n = int(n_compounds)
        self.base = int(compound_base)
        self.dir = 1 if direction == "max" else -1
        dev = _require_cuda(device)
        self.keys = torch.full((max(self.n, 1),), -1, dtype=torch.int64, device=dev)   # all-ones

    def update(self, compound, pose_id, scores):
        N.check(N.lib().fs_best_pose_update(_ptr(compound), self.base, _ptr(pose_id), _ptr(scores), scores.numel(),
                                            self.n, self.dir, _ptr(self.keys), _stream()), "fs_best_pose_update")

    def result(self):
        s = torch.empty(max(self.n, 1), dtype=torch.float32, device=self.keys.device)
        p = torch.empty(max(self.n, 1), dtype=torch.int64, device=self.keys.device)
        N.check(N.lib().fs_best_pose_decode(_ptr(self.keys), self.n, self.dir, _ptr(s), _ptr(p), _stream()),
                "fs_best_pose_decode")
        return s[: self.n], p[: self.n]
