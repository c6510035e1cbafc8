"""C-ABI library: builds, loads, exports every declared symbol.  CPU only
(no compute calls: this container has no GPU)."""

import ctypes as C
import os
import re

import pytest

from paper_2104_04547_b200 import _native as N
from paper_2104_04547_b200 import engine as E
from tests._cfg import COHERENT, GRAPH, TOY_FUSION, TOY_GRAPH, TOY_VOXEL, VOXEL

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fusionb200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(N.LIB_PATH):
        from paper_2104_04547_b200 import build_native
        build_native.build()
    return N.lib()


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(N.EXPORTS) == names


def test_status_strings_and_version(lib):
    assert lib.fs_strerror(0) == b"ok"
    assert b"invalid" in lib.fs_strerror(N.FS_EINVAL)
    assert lib.fs_version() >= 100


def test_weights_bytes_default_and_toy(lib):
    d = E.model_desc(VOXEL, GRAPH, COHERENT)
    n = lib.fs_weights_bytes(C.byref(d))
    # fp32 copy of the 758,465 voxel-head params at least (GRU message weights
    # are folded into the gate matrices, so the graph head packs smaller)
    assert n >= 758_465 * 4
    t = E.model_desc(TOY_VOXEL, TOY_GRAPH, TOY_FUSION, box_size=8.0)
    assert 0 < lib.fs_weights_bytes(C.byref(t)) < n


def test_invalid_desc_rejected(lib):
    bad = dict(GRAPH, k_cov=9)
    d = E.model_desc(VOXEL, bad, COHERENT)
    assert lib.fs_weights_bytes(C.byref(d)) == 0
    d = E.model_desc(VOXEL, dict(GRAPH, cov_thresh=6.0), COHERENT)
    assert lib.fs_weights_bytes(C.byref(d)) == 0
    d = E.model_desc(dict(VOXEL, grid_extent=4), GRAPH, COHERENT)
    assert lib.fs_weights_bytes(C.byref(d)) == 0


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="CUDA"):
        E.batch_from_arrays([[0.0, 0.0, 0.0]], [0], [0], [0, 1])
