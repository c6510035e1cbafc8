"""ctypes loader of oracle/radius_graph.c -- TEST INFRASTRUCTURE ONLY.

Batched exact radius graph on the host (restates complexes.py:237-246; see the
C file's header).  Built with gcc on first use into oracle/_build/ (git-ignored;
the .so travels to the GPU box with the snapshot, and is rebuilt there if
missing -- gcc is in the same image).  Only tests/, smoke() and bench.py's
CPU legs may use it.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "radius_graph.c")
LIB = os.path.join(HERE, "_build", "libradius_oracle.so")
# -ffp-contract=off: the predicate is ((dx*dx + dy*dy) + dz*dz) with every
# product rounded, exactly as numpy/scipy evaluate it
CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math"]

_lib = None


def build(force=False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        tmp = LIB + f".{os.getpid()}.tmp"
        subprocess.run(["gcc", *CFLAGS, SRC, "-o", tmp, "-lm"], check=True)
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        h = C.CDLL(build())
        p = C.c_void_p
        h.rg_count.argtypes = [p, p, p, C.c_int64, C.c_double, C.c_double, p, p]
        h.rg_fill.argtypes = [p, p, p, C.c_int64, C.c_double, C.c_double, p, p, p, p, p, p]
        h.rg_count.restype = h.rg_fill.restype = None
        _lib = h
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data)


def radius_pairs_batch(xyz, roles, atom_off, cov_thresh=2.24, noncov_thresh=5.22):
    """Edges of every pose.  Returns (cov_ij [Ec,2], cov_d [Ec], cov_off [P+1],
    ncov_ij [En,2], ncov_d [En], ncov_off [P+1]); pose p's edges are rows
    off[p]..off[p+1], pose-local node ids, lexsorted by (i, j)."""
    xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    roles = np.ascontiguousarray(roles, dtype=np.int64)
    atom_off = np.ascontiguousarray(atom_off, dtype=np.int64)
    P = len(atom_off) - 1
    nc = np.zeros(P, dtype=np.int64)
    nn = np.zeros(P, dtype=np.int64)
    L = lib()
    L.rg_count(_p(xyz), _p(roles), _p(atom_off), P, cov_thresh, noncov_thresh, _p(nc), _p(nn))
    coff = np.concatenate([[0], np.cumsum(nc)]).astype(np.int64)
    noff = np.concatenate([[0], np.cumsum(nn)]).astype(np.int64)
    cij = np.zeros((max(int(coff[-1]), 1), 2), dtype=np.int64)
    cd = np.zeros(max(int(coff[-1]), 1))
    nij = np.zeros((max(int(noff[-1]), 1), 2), dtype=np.int64)
    nd = np.zeros(max(int(noff[-1]), 1))
    L.rg_fill(_p(xyz), _p(roles), _p(atom_off), P, cov_thresh, noncov_thresh, _p(coff), _p(noff), _p(cij), _p(cd),
              _p(nij), _p(nd))
    return cij[: coff[-1]], cd[: coff[-1]], coff, nij[: noff[-1]], nd[: noff[-1]], noff


def radius_pairs(positions, roles, cov_thresh=2.24, noncov_thresh=5.22):
    """One pose; same return convention as fusion_oracle.radius_pairs."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    ce, cd, _, ne, nd, _ = radius_pairs_batch(pos, roles, np.array([0, len(pos)]), cov_thresh, noncov_thresh)
    return ce, cd, ne, nd
