"""Packed pose library format: CPU round trip."""

import numpy as np
import pytest

from paper_2104_04547_b200 import poselib, synth


def _lib():
    pockets = [synth.make_pocket(300, seed=3, name="a"), synth.make_pocket(120, seed=4, name="b")]
    lib = synth.concat([synth.make_poses(5, 3, seed=5, target=0),
                        synth.make_poses(4, 2, seed=6, target=1, compound_base=5)])
    return pockets, lib


def test_roundtrip_is_exact(tmp_path):
    pockets, lib = _lib()
    path = tmp_path / "lib.fspl"
    poselib.save_library(path, pockets, lib)
    pk2, lib2 = poselib.load_library(path)
    assert len(pk2) == 2
    for a, b in zip(pockets, pk2):
        assert np.array_equal(a.xyz, b.xyz) and np.array_equal(a.elem, b.elem) and np.array_equal(a.role, b.role)
    for f in ("xyz", "elem", "role", "atom_off", "target", "compound", "pose_id"):
        assert np.array_equal(getattr(lib, f), getattr(lib2, f)), f
    assert lib2.n_poses == lib.n_poses


def test_sections_are_aligned_and_mapped(tmp_path):
    pockets, lib = _lib()
    path = tmp_path / "lib.fspl"
    poselib.save_library(path, pockets, lib)
    _, lib2 = poselib.load_library(path)
    assert isinstance(lib2.xyz.base, (np.memmap, np.ndarray))       # a view, no parse
    assert not lib2.xyz.flags.writeable
    raw = np.fromfile(path, dtype=np.uint8)
    off = lib2.xyz.ctypes.data - np.asarray(lib2.atom_off).ctypes.data
    assert off > 0 and raw[:8].tobytes() == poselib.MAGIC


def test_rejects_foreign_file(tmp_path):
    path = tmp_path / "x.bin"
    path.write_bytes(b"NOTALIB!" + b"\0" * 64)
    with pytest.raises(ValueError, match="not a packed pose library"):
        poselib.load_library(path)


def test_empty_library(tmp_path):
    pockets, lib = _lib()
    empty = lib.slice(0, 0)
    path = tmp_path / "e.fspl"
    poselib.save_library(path, pockets, empty)
    _, lib2 = poselib.load_library(path)
    assert lib2.n_poses == 0 and lib2.atom_off.tolist() == [0]
