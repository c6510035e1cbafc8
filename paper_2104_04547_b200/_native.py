"""ctypes binding of libfusionb200.so (the C-ABI in include/fusionb200.h).

There is no CPU fallback: if the in-tree library is missing or a CUDA device
is absent, the product path raises.  Torch is used only as the allocator of
device memory and for streams; every computation is a call through this ABI.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FS_LIB: an alternative in-tree build (A/B kernel experiments)
LIB_PATH = os.environ.get("FS_LIB") or os.path.join(HERE, "libfusionb200.so")

FS_OK, FS_EINVAL, FS_ECAPACITY, FS_ECUDA, FS_ENOTSUP = 0, -1, -2, -3, -4
FS_ERR_ROLE, FS_ERR_NAN, FS_ERR_NONFINITE, FS_ERR_EDGE_CAP, FS_ERR_TOO_LARGE = 1, 2, 4, 8, 16
FS_ERR_GRID_NONFINITE, FS_ERR_FEAT_NONFINITE, FS_ERR_NOT_FACTORED = 32, 64, 128
FS_MAX_POSE_ATOMS = 4096
FS_PREC_FP32, FS_PREC_BF16, FS_PREC_MIXED = 0, 1, 2
FS_GRID_NCDHW_F64, FS_GRID_NDHWC_F32, FS_GRID_NDHWC_BF16 = 0, 1, 2
FS_MODE_LATE, FS_MODE_MID, FS_MODE_COHERENT = 0, 1, 2

STAGES = ("featurize", "conv1", "conv2", "conv3", "conv4", "dense", "gnn", "fusion", "end")
PRECISIONS = {"fp32": FS_PREC_FP32, "bf16": FS_PREC_BF16, "mixed": FS_PREC_MIXED}

# every symbol include/fusionb200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "fs_strerror", "fs_version", "fs_last_cuda_error", "fs_launch_count", "fs_set_stage_events", "fs_set_overlap",
    "fs_weights_bytes", "fs_model_create",
    "fs_model_destroy", "fs_model_supports", "fs_node_offsets", "fs_node_offsets_ws_bytes",
    "fs_voxelize", "fs_node_features", "fs_graph_count", "fs_graph_rows", "fs_graph_rows_ws_bytes",
    "fs_graph_fill", "fs_graph_edge_counts", "fs_graph_edges", "fs_workspace_bytes", "fs_features_workspace_bytes",
    "fs_score_poses", "fs_score_features", "fs_debug_conv", "fs_topk_ws_bytes", "fs_topk_merge",
    "fs_best_pose", "fs_best_pose_update", "fs_best_pose_decode",
    "fs_pocket_cache_bytes", "fs_pocket_prepare_ws_bytes", "fs_pocket_prepare", "fs_score_poses_cached",
    "fs_scoring_graph_ws_bytes", "fs_scoring_graph",
)


class PoseBatchC(C.Structure):
    _fields_ = [
        ("pocket_xyz", C.c_void_p), ("pocket_elem", C.c_void_p), ("pocket_role", C.c_void_p),
        ("pocket_off", C.c_void_p), ("n_pockets", C.c_int32),
        ("atom_xyz", C.c_void_p), ("atom_elem", C.c_void_p), ("atom_role", C.c_void_p),
        ("atom_off", C.c_void_p), ("pose_target", C.c_void_p), ("n_poses", C.c_int32),
        ("max_pose_atoms", C.c_int32),
    ]


class ModelDescC(C.Structure):
    _fields_ = [
        ("grid_extent", C.c_int32), ("in_channels", C.c_int32), ("conv_filters_1", C.c_int32),
        ("conv_filters_2", C.c_int32), ("dense_nodes", C.c_int32), ("kernel_1", C.c_int32),
        ("kernel_2", C.c_int32), ("residual_1", C.c_int32), ("residual_2", C.c_int32),
        ("batch_norm", C.c_int32), ("c_elem", C.c_int32), ("k_cov", C.c_int32),
        ("k_noncov", C.c_int32), ("gather_width_cov", C.c_int32),
        ("gather_width_noncov", C.c_int32), ("cov_thresh", C.c_double),
        ("noncov_thresh", C.c_double), ("box_size", C.c_double), ("fusion_mode", C.c_int32),
        ("n_fusion_layers", C.c_int32), ("model_specific_layers", C.c_int32),
        ("residual_fusion", C.c_int32), ("activation", C.c_int32),
        ("fusion_dense_nodes", C.c_int32),
    ]


class NativeError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        msg = f"{where}: {lib().fs_strerror(code).decode()} ({code})"
        if code == FS_ECUDA:
            msg += f": {lib().fs_last_cuda_error().decode()}"
        super().__init__(msg)


_LIB = None

_P, _I32, _I64, _SZ, _D = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t, C.c_double


def _sig(lib):
    sp = C.POINTER(PoseBatchC)
    md = C.POINTER(ModelDescC)
    t = {
        "fs_strerror": (C.c_char_p, [C.c_int]),
        "fs_version": (C.c_int, []),
        "fs_last_cuda_error": (C.c_char_p, []),
        "fs_launch_count": (C.c_longlong, []),
        "fs_set_stage_events": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
        "fs_set_overlap": (C.c_int, [C.c_int]),
        "fs_weights_bytes": (_SZ, [md]),
        "fs_model_create": (C.c_int, [md, C.POINTER(C.c_char_p), C.POINTER(C.c_void_p), C.c_int,
                                      _P, _SZ, _P, C.POINTER(C.c_void_p)]),
        "fs_model_destroy": (C.c_int, [_P]),
        "fs_model_supports": (C.c_int, [_P, C.c_int]),
        "fs_node_offsets": (C.c_int, [sp, _P, _P, _SZ, _P]),
        "fs_node_offsets_ws_bytes": (_SZ, [_I32]),
        "fs_voxelize": (C.c_int, [sp, _I32, _I32, _D, _I32, _P, _P, _P]),
        "fs_node_features": (C.c_int, [sp, _P, _I32, _D, _P, _P]),
        "fs_graph_count": (C.c_int, [sp, _P, _D, _D, _P, _P, _P, _P]),
        "fs_graph_rows": (C.c_int, [_P, _I64, _P, _P, _SZ, _P]),
        "fs_graph_rows_ws_bytes": (_SZ, [_I64]),
        "fs_graph_fill": (C.c_int, [sp, _P, _D, _D, _P, _P, _P, _P, _P, _P, _I64, _I64, _P, _P]),
        "fs_graph_edge_counts": (C.c_int, [_P, _I32, _P, _P, _P, _P, _SZ, _P]),
        "fs_graph_edges": (C.c_int, [_P, _I32, _P, _P, _P, _P, _P, _P, _P]),
        "fs_workspace_bytes": (_SZ, [_P, _I32, _I64, _I64, C.c_int]),
        "fs_features_workspace_bytes": (_SZ, [_P, _I32, _I64, _I32, _I64, C.c_int]),
        "fs_scoring_graph_ws_bytes": (_SZ, [_I32, _I32, _I64, _I32, _I32]),
        "fs_scoring_graph": (C.c_int, [sp, _D, _D, _I64, _I32, _I32, _I32, _D, _P, _SZ, _P, _P, _P, _P, _P, _P,
                                       _P, _P]),
        "fs_score_poses": (C.c_int, [_P, C.c_int, sp, _I64, _P, _SZ, _P, _P, _P, _P, _P, _P, _P]),
        "fs_pocket_cache_bytes": (_SZ, [_P, _I32]),
        "fs_pocket_prepare_ws_bytes": (_SZ, [_P, _I32, _I32]),
        "fs_pocket_prepare": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, _I32, _I32, _P, _P, _P, _SZ, _P]),
        "fs_score_poses_cached": (C.c_int, [_P, C.c_int, sp, _P, _I32, _I64, _P, _SZ, _P, _P, _P, _P, _P, _P,
                                            _P]),
        "fs_score_features": (C.c_int, [_P, C.c_int, _I32, _P, _P, _P, _I64, _I32, _P, _I64, _P, _I64,
                                        _I32, _P, _SZ, _P, _P, _P, _P, _P, _P, _P]),
        "fs_debug_conv": (C.c_int, [_P, C.c_int, _I32, _P, _P, _P, _P]),
        "fs_topk_ws_bytes": (_SZ, [_I64]),
        "fs_topk_merge": (C.c_int, [_P, _P, _I64, _P, _P, _I64, _I32, _P, _P, _P, _SZ, _P]),
        "fs_best_pose": (C.c_int, [_P, _P, _P, _I64, _I64, _I32, _P, _P, _P]),
        "fs_best_pose_update": (C.c_int, [_P, _I64, _P, _P, _I64, _I64, _I32, _P, _P]),
        "fs_best_pose_decode": (C.c_int, [_P, _I64, _I32, _P, _P, _P]),
    }
    for name, (res, args) in t.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args


def lib():
    """Load the in-tree library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} missing: build it with `python -m paper_2104_04547_b200.build_native` "
                "(there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        _sig(handle)
        _LIB = handle
    return _LIB


def check(rc, where):
    if rc != FS_OK:
        raise NativeError(rc, where)
