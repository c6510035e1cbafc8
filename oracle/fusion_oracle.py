"""CPU oracle for the Coherent-Fusion pose-scoring path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it;
the package ``paper_2104_04547_b200`` must never route work through it (its
CUDA library fails loudly instead).

It is an independent float64 numpy restatement of the reference algorithm
(``fusionscreen``, mounted read-only at /root/reference/pkg/src).  Each
function cites the reference file:line it restates.  Parity status: PINNED --
``tests/test_oracle_golden.py`` checks every function here against golden
vectors produced by importing the unmodified reference in the build container
(``tests/golden/make_golden.py``; fixtures committed under ``tests/golden/``).

Third-party arithmetic the reference relies on, restated here:
  * scipy ``cKDTree.query_pairs(r)`` (scipy 1.18.1 in this image): a pair is
    reported iff the float64 sum ((dx*dx + dy*dy) + dz*dz) <= r*r.  Verified
    here on 400k pairs placed within 3 ulp of r ("radius
    predicate").  ``build_graph`` then keeps pairs by ``np.linalg.norm`` which
    equals sqrt of the same sum, bitwise.
  * numpy ``einsum``/``@`` on OpenBLAS: plain float64 dot products; restated
    with ``np.tensordot`` (summation order differs => ~1e-15 relative).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from numpy.lib.stride_tricks import sliding_window_view

PROTEIN, LIGAND = 0, 1                       # complexes.py:26
SELU_ALPHA = 1.6732632423543772              # autodiff.py:28
SELU_LAMBDA = 1.0507009873554805             # autodiff.py:29
LEAKY_SLOPE = 0.01                           # autodiff.py:30
THRESHOLD_RANGE = (1.2, 5.9)                 # complexes.py:207


def _g(cfg, name):
    """Config field accessor that works for dataclasses and dicts."""
    return cfg[name] if isinstance(cfg, dict) else getattr(cfg, name)


# ---------------------------------------------------------------------------
# featurization
# ---------------------------------------------------------------------------

def voxelize(positions, elements, roles, extent=16, c_elem=4, box_size=16.0):
    """Nearest-voxel count splat.  Restates complexes.py:171-184.

    idx = clip(floor(((pos + box/2) / box) * G), 0, G-1) in float64, channel =
    role*c_elem + clip(elem, 0, c_elem-1); every atom adds 1.0.
    Returns float64 [2*c_elem, G, G, G] with axes (C, x, y, z).
    """
    if extent < 8:
        raise ValueError(f"grid extent must be >= 8, got {extent}")
    pos = np.asarray(positions, dtype=np.float64)
    g = int(extent)
    cell = np.floor((pos + box_size / 2.0) / box_size * g)
    cell = np.clip(cell, 0, g - 1).astype(np.int64)
    chan = np.asarray(roles, dtype=np.int64) * c_elem + np.clip(
        np.asarray(elements, dtype=np.int64), 0, c_elem - 1)
    flat = ((chan * g + cell[:, 0]) * g + cell[:, 1]) * g + cell[:, 2]
    occ = np.bincount(flat, minlength=2 * c_elem * g ** 3).astype(np.float64)
    return occ.reshape(2 * c_elem, g, g, g)


def node_features(positions, elements, roles, c_elem=4, box_size=16.0):
    """[one-hot(clip elem) | role | pos/box + 0.5].  Restates complexes.py:233-236."""
    pos = np.asarray(positions, dtype=np.float64)
    n = len(pos)
    f = np.zeros((n, c_elem + 4))
    f[np.arange(n), np.clip(np.asarray(elements, dtype=np.int64), 0, c_elem - 1)] = 1.0
    f[:, c_elem] = np.asarray(roles, dtype=np.float64)
    f[:, c_elem + 1:] = pos / box_size + 0.5
    return f


def radius_pairs(positions, roles, cov_thresh=2.24, noncov_thresh=5.22):
    """Exact edge predicate of complexes.py:237-246, canonical order.

    Candidate pairs i<j come from the kd-tree radius query at
    r = max(cov, noncov) (predicate: d2 <= r*r, d2 = (dx^2+dy^2)+dz^2);
    d = sqrt(d2) (== np.linalg.norm bitwise); covalent = same role and
    d <= cov; non-covalent = different role and d <= noncov.
    Returns (cov_edges[e,2], cov_d[e], ncov_edges[e,2], ncov_d[e]) with rows
    lexsorted by (i, j) -- the reference emits kd-tree traversal order, so
    comparisons against it lexsort first.
    """
    lo, hi = THRESHOLD_RANGE
    for t in (cov_thresh, noncov_thresh):
        if not lo <= t <= hi:
            raise ValueError(f"threshold {t} outside searched range [{lo}, {hi}]")
    pos = np.asarray(positions, dtype=np.float64)
    roles = np.asarray(roles)
    n = len(pos)
    r = max(cov_thresh, noncov_thresh)
    r2 = r * r
    cov_i, cov_j, cov_d, nc_i, nc_j, nc_d = [], [], [], [], [], []
    block = 512
    for s in range(0, n, block):
        ii = np.arange(s, min(n, s + block))
        diff = pos[ii, None, :] - pos[None, :, :]
        d2 = (diff[..., 0] * diff[..., 0] + diff[..., 1] * diff[..., 1]) \
            + diff[..., 2] * diff[..., 2]
        upper = np.arange(n)[None, :] > ii[:, None]
        cand = upper & (d2 <= r2)
        a, b = np.nonzero(cand)
        if not len(a):
            continue
        gi, gj = ii[a], b
        d = np.sqrt(d2[a, b])
        same = roles[gi] == roles[gj]
        m_c = same & (d <= cov_thresh)
        m_n = ~same & (d <= noncov_thresh)
        cov_i.append(gi[m_c]); cov_j.append(gj[m_c]); cov_d.append(d[m_c])
        nc_i.append(gi[m_n]); nc_j.append(gj[m_n]); nc_d.append(d[m_n])

    def pack(i, j, d):
        if not i:
            return np.zeros((0, 2), dtype=np.int64), np.zeros(0)
        i, j, d = np.concatenate(i), np.concatenate(j), np.concatenate(d)
        order = np.lexsort((j, i))
        return np.stack([i[order], j[order]], axis=1).astype(np.int64), d[order]

    ce, cd = pack(cov_i, cov_j, cov_d)
    ne, nd = pack(nc_i, nc_j, nc_d)
    return ce, cd, ne, nd


def canonical_edges(edges, dists):
    """Lexsort an (i<j) edge list and its distances by (i, j)."""
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    dists = np.asarray(dists, dtype=np.float64)
    if not len(edges):
        return edges, dists
    order = np.lexsort((edges[:, 1], edges[:, 0]))
    return edges[order], dists[order]


def adjacency(n, edges):
    """Symmetric 0/1 adjacency from i<j pairs.  Restates models.py:238-247."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    rows = np.concatenate([e[:, 0], e[:, 1]])
    cols = np.concatenate([e[:, 1], e[:, 0]])
    return sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(n, n))


# ---------------------------------------------------------------------------
# parameter initialisation (scaled uniform fan-in, one RNG in fixed order)
# ---------------------------------------------------------------------------

def _uniform(rng, fan_in, shape):
    bound = 1.0 / np.sqrt(max(fan_in, 1))                  # models.py:145-147
    return rng.uniform(-bound, bound, size=shape)


def init_params(vcfg, gcfg, fcfg, seed=0):
    """Same draw order as FusionModel.__init__ (models.py:415-428):
    voxel (models.py:150-172), graph (:175-198), fusion (:201-218)."""
    rng = np.random.default_rng(seed)
    k1, k2 = _g(vcfg, "kernel_1"), _g(vcfg, "kernel_2")
    c, f1, f2 = _g(vcfg, "in_channels"), _g(vcfg, "conv_filters_1"), _g(vcfg, "conv_filters_2")
    dn = _g(vcfg, "dense_nodes")
    flat = f2 * (_g(vcfg, "grid_extent") // 4) ** 3
    lat_v = dn // 2
    v = {}
    for name, fan, shape in (
            ("conv1_w", c * k1 ** 3, (f1, c, k1, k1, k1)), ("conv1_b", c * k1 ** 3, f1),
            ("conv2_w", f1 * k2 ** 3, (f1, f1, k2, k2, k2)), ("conv2_b", f1 * k2 ** 3, f1),
            ("conv3_w", f1 * k2 ** 3, (f2, f1, k2, k2, k2)), ("conv3_b", f1 * k2 ** 3, f2),
            ("conv4_w", f2 * k2 ** 3, (f2, f2, k2, k2, k2)), ("conv4_b", f2 * k2 ** 3, f2),
            ("dense1_w", flat, (flat, dn)), ("dense1_b", flat, dn),
            ("dense2_w", dn, (dn, lat_v)), ("dense2_b", dn, lat_v),
            ("out_w", lat_v, (lat_v, 1)), ("out_b", lat_v, 1)):
        v[name] = _uniform(rng, fan, shape)
    if _g(vcfg, "batch_norm"):
        v["bn1_gamma"], v["bn1_beta"] = np.ones(f1), np.zeros(f1)
        v["bn2_gamma"], v["bn2_beta"] = np.ones(f2), np.zeros(f2)
    d, gn = _g(gcfg, "gather_width_cov"), _g(gcfg, "gather_width_noncov")
    fw = _g(gcfg, "c_elem") + 4
    gp = {"embed_w": _uniform(rng, fw, (fw, d)), "embed_b": _uniform(rng, fw, d),
          "gather_gate_w": _uniform(rng, d, (d, gn)), "gather_gate_b": _uniform(rng, d, gn),
          "gather_feat_w": _uniform(rng, d, (d, gn)), "gather_feat_b": _uniform(rng, d, gn)}
    for phase in ("cov", "noncov"):
        gp[f"{phase}_msg_w"] = _uniform(rng, d, (d, d))
        for gate in "zrh":
            gp[f"{phase}_w{gate}"] = _uniform(rng, d, (d, d))
            gp[f"{phase}_u{gate}"] = _uniform(rng, d, (d, d))
            gp[f"{phase}_b{gate}"] = _uniform(rng, d, d)
    w1 = int(gn / 1.5)
    w2 = w1 // 2
    gp["dense1_w"], gp["dense1_b"] = _uniform(rng, gn, (gn, w1)), _uniform(rng, gn, w1)
    gp["dense2_w"], gp["dense2_b"] = _uniform(rng, w1, (w1, w2)), _uniform(rng, w1, w2)
    gp["out_w"], gp["out_b"] = _uniform(rng, w2, (w2, 1)), _uniform(rng, w2, 1)
    fp = {}
    if _g(fcfg, "mode") != "late":
        width = gn + lat_v
        if _g(fcfg, "model_specific_layers"):
            fp["ms_graph_w"], fp["ms_graph_b"] = _uniform(rng, gn, (gn, gn)), _uniform(rng, gn, gn)
            fp["ms_voxel_w"], fp["ms_voxel_b"] = (_uniform(rng, lat_v, (lat_v, lat_v)),
                                                  _uniform(rng, lat_v, lat_v))
            width *= 2
        nl, fd = _g(fcfg, "n_fusion_layers"), _g(fcfg, "fusion_dense_nodes")
        widths = [width] + [fd] * (nl - 1) + [1]
        for i in range(nl):
            fp[f"fuse{i}_w"] = _uniform(rng, widths[i], (widths[i], widths[i + 1]))
            fp[f"fuse{i}_b"] = _uniform(rng, widths[i], widths[i + 1])
    return v, gp, fp


# ---------------------------------------------------------------------------
# float64 forward
# ---------------------------------------------------------------------------

def sigmoid(x):
    return 0.5 * (1.0 + np.tanh(0.5 * x))            # autodiff.py:322-327


def activation(kind, x):
    if kind == "relu":                                # autodiff.py:298-300
        return np.maximum(x, 0.0)
    if kind == "leaky-relu":                          # autodiff.py:303-308
        return np.where(x > 0, x, LEAKY_SLOPE * x)
    if kind == "selu":                                # autodiff.py:311-319
        return SELU_LAMBDA * np.where(x > 0, x, SELU_ALPHA * np.expm1(x))
    raise ValueError(kind)


def conv3d(x, w, b):
    """Cross-correlation, stride 1, zero pad k//2.  Restates autodiff.py:208-232.

    x [C,D,H,W] (one pose), w [O,C,k,k,k] -> [O,D,H,W].
    """
    k = w.shape[2]
    p = k // 2
    xp = np.pad(x, ((0, 0), (p, p), (p, p), (p, p)))
    win = sliding_window_view(xp, (k, k, k), axis=(1, 2, 3))   # [C,D,H,W,k,k,k]
    out = np.tensordot(win, w, axes=([0, 4, 5, 6], [1, 2, 3, 4]))  # [D,H,W,O]
    return np.moveaxis(out, -1, 0) + b[:, None, None, None]


def maxpool3d(x, s=2):
    """Non-overlapping s^3 max.  Restates autodiff.py:251-269."""
    c, d, h, w = x.shape
    return x.reshape(c, d // s, s, h // s, s, w // s, s).max(axis=(2, 4, 6))


def batch_norm_eval(x, gamma, beta, state=None, eps=1e-5):
    """Eval-mode batch norm over channel axis 0.  Restates autodiff.py:335-368."""
    c = x.shape[0]
    mean = np.zeros(c) if state is None else state["mean"]
    var = np.ones(c) if state is None else state["var"]
    shape = (c,) + (1,) * (x.ndim - 1)
    inv = 1.0 / np.sqrt(var + eps)
    return gamma.reshape(shape) * ((x - mean.reshape(shape)) * inv.reshape(shape)) \
        + beta.reshape(shape)


def voxel_head(vp, vcfg, grid, bn_state=None):
    """One pose.  Restates models.py:285-322 in eval mode.  Returns (pred, latent[64])."""
    bn_state = bn_state or {}
    use_bn = _g(vcfg, "batch_norm")
    h1 = activation("relu", conv3d(grid, vp["conv1_w"], vp["conv1_b"]))
    if use_bn:
        h1 = batch_norm_eval(h1, vp["bn1_gamma"], vp["bn1_beta"], bn_state.get("bn1"))
    h2 = activation("relu", conv3d(h1, vp["conv2_w"], vp["conv2_b"]))
    if _g(vcfg, "residual_1"):
        h2 = h2 + h1
    h2 = maxpool3d(h2)
    h3 = activation("relu", conv3d(h2, vp["conv3_w"], vp["conv3_b"]))
    if use_bn:
        h3 = batch_norm_eval(h3, vp["bn2_gamma"], vp["bn2_beta"], bn_state.get("bn2"))
    h4 = activation("relu", conv3d(h3, vp["conv4_w"], vp["conv4_b"]))
    if _g(vcfg, "residual_2"):
        h4 = h4 + h3
    flat = maxpool3d(h4).reshape(-1)                   # (C, D, H, W) order, autodiff.py:549-553
    d1 = activation("relu", flat @ vp["dense1_w"] + vp["dense1_b"])
    d2 = activation("relu", d1 @ vp["dense2_w"] + vp["dense2_b"])
    pred = d2 @ vp["out_w"] + vp["out_b"]
    return float(pred[0]), d2


def graph_head(gp, gcfg, feats, adj_cov, adj_ncov):
    """One pose.  Restates models.py:334-371.  Returns (pred, latent[gn])."""
    h = np.tanh(feats @ gp["embed_w"] + gp["embed_b"])
    for phase, adj, steps in (("cov", adj_cov, _g(gcfg, "k_cov")),
                              ("noncov", adj_ncov, _g(gcfg, "k_noncov"))):
        w = {k: gp[f"{phase}_{k}"] for k in
             ("msg_w", "wz", "wr", "wh", "uz", "ur", "uh", "bz", "br", "bh")}
        for _ in range(steps):
            m = np.asarray(adj @ (h @ w["msg_w"]))
            z = sigmoid(m @ w["wz"] + w["bz"] + h @ w["uz"])
            r = sigmoid(m @ w["wr"] + w["br"] + h @ w["ur"])
            hh = np.tanh(m @ w["wh"] + w["bh"] + (r * h) @ w["uh"])
            h = h + z * (hh - h)
    gates = sigmoid(h @ gp["gather_gate_w"] + gp["gather_gate_b"])
    vals = np.tanh(h @ gp["gather_feat_w"] + gp["gather_feat_b"])
    latent = (gates * vals).mean(axis=0)                # pool rows are 1/n, models.py:249-254
    d1 = activation("relu", latent @ gp["dense1_w"] + gp["dense1_b"])
    d2 = activation("relu", d1 @ gp["dense2_w"] + gp["dense2_b"])
    pred = d2 @ gp["out_w"] + gp["out_b"]
    return float(pred[0]), latent


def fusion_head(fp, fcfg, lat_g, lat_v):
    """Restates models.py:374-396 (eval mode, dropout identity)."""
    act = _g(fcfg, "activation")
    parts = [lat_g, lat_v]
    if _g(fcfg, "model_specific_layers"):
        parts.append(activation(act, lat_g @ fp["ms_graph_w"] + fp["ms_graph_b"]))
        parts.append(activation(act, lat_v @ fp["ms_voxel_w"] + fp["ms_voxel_b"]))
    h = np.concatenate(parts)
    n = _g(fcfg, "n_fusion_layers")
    prev = None
    for i in range(n - 1):
        h = activation(act, h @ fp[f"fuse{i}_w"] + fp[f"fuse{i}_b"])
        if _g(fcfg, "residual_fusion") and prev is not None:
            h = h + prev
        prev = h
    return float((h @ fp[f"fuse{n - 1}_w"] + fp[f"fuse{n - 1}_b"])[0])


def score_pose(params, cfgs, positions, elements, roles, box_size=16.0, bn_state=None):
    """Featurize + both heads + fusion for one complex (models.py:638-651, :470-498).

    Returns dict(score, lat_v, lat_g, pred_v, pred_g, grid, cov, ncov).
    """
    vp, gp, fp = params
    vcfg, gcfg, fcfg = cfgs
    grid = voxelize(positions, elements, roles, _g(vcfg, "grid_extent"),
                    _g(vcfg, "in_channels") // 2, box_size)
    ce, cd, ne, nd = radius_pairs(positions, roles, _g(gcfg, "cov_thresh"),
                                  _g(gcfg, "noncov_thresh"))
    n = len(positions)
    feats = node_features(positions, elements, roles, _g(gcfg, "c_elem"), box_size)
    pv, lat_v = voxel_head(vp, vcfg, grid, bn_state)
    pg, lat_g = graph_head(gp, gcfg, feats, adjacency(n, ce), adjacency(n, ne))
    if _g(fcfg, "mode") == "late":
        score = (pv + pg) / 2.0                              # models.py:399-405
    else:
        score = fusion_head(fp, fcfg, lat_g, lat_v)
    return dict(score=score, lat_v=lat_v, lat_g=lat_g, pred_v=pv, pred_g=pg,
                grid=grid, cov=(ce, cd), ncov=(ne, nd))


# ---------------------------------------------------------------------------
# ranking
# ---------------------------------------------------------------------------

def topk(scores, k, index_base=0):
    """Top-k by (score desc, global pose index asc) -- the tie rule of
    evaluate.aggregate_best_pose (evaluate.py:67-83) applied to ranking."""
    s = np.asarray(scores)
    idx = np.arange(len(s), dtype=np.int64) + index_base
    order = np.lexsort((idx, -s.astype(np.float64)))[:k]
    return s[order], idx[order]


def best_pose(compound, target, pose_id, score, direction="max"):
    """Restates evaluate.aggregate_best_pose (evaluate.py:67-83)."""
    if direction not in ("max", "min"):
        raise ValueError(f"direction must be max or min, got {direction!r}")
    sign = 1.0 if direction == "max" else -1.0
    best = {}
    for c, t, p, s in zip(compound, target, pose_id, score):
        cand = (-sign * s, p)
        if (c, t) not in best or cand < best[(c, t)]:
            best[(c, t)] = cand
    return {k: (p, -sign * ns) for k, (ns, p) in best.items()}
