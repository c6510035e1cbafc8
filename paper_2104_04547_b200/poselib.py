"""Binary packed pose library + pinned streaming loader.

The reference reads screening libraries from JSON lines
(complexes.load_dataset, complexes.py:309-329) and featurizes them on the host
before scoring (cli.py:250-256) -- the paper's stated bottleneck
(PAPER.md:322).  Here a library is one flat little-endian file that maps
straight onto the device batch layout (fs_pose_batch):

    header  : magic b"FSPLIB01", u64 n_pockets, u64 n_pocket_atoms, u64 n_poses, u64 n_atoms
    pockets : i64 pocket_off[n_pockets+1]
              f64 pocket_xyz[n_pocket_atoms*3], i32 pocket_elem[.], i32 pocket_role[.]
    poses   : i64 atom_off[n_poses+1], i32 target[n_poses], i64 compound[n_poses],
              i64 pose_id[n_poses], f64 xyz[n_atoms*3], i32 elem[n_atoms], i32 role[n_atoms]

Every section is 64-byte aligned.  ``load_library`` memory-maps the file (no
parse, no copy); ``StreamingLoader`` walks it batch by batch through a
double-buffered pinned host staging area and a dedicated copy stream, so the
host->device transfer of batch i+1 overlaps the scoring of batch i.
"""

from __future__ import annotations

import numpy as np

from .synth import Pocket, PoseLibrary

MAGIC = b"FSPLIB01"
_ALIGN = 64


def _pad(f):
    pos = f.tell()
    if pos % _ALIGN:
        f.write(b"\0" * (_ALIGN - pos % _ALIGN))


def save_library(path, pockets, lib: PoseLibrary) -> None:
    p_off = np.concatenate([[0], np.cumsum([len(p.xyz) for p in pockets])]).astype(np.int64)
    with open(path, "wb") as f:
        f.write(MAGIC)
        np.array([len(pockets), p_off[-1], lib.n_poses, lib.atom_off[-1]], dtype="<u8").tofile(f)
        for arr in (p_off,
                    np.concatenate([p.xyz for p in pockets]).astype("<f8"),
                    np.concatenate([p.elem for p in pockets]).astype("<i4"),
                    np.concatenate([p.role for p in pockets]).astype("<i4"),
                    lib.atom_off.astype("<i8"), lib.target.astype("<i4"), lib.compound.astype("<i8"),
                    lib.pose_id.astype("<i8"), lib.xyz.astype("<f8"), lib.elem.astype("<i4"),
                    lib.role.astype("<i4")):
            _pad(f)
            np.ascontiguousarray(arr).tofile(f)


def load_library(path):
    """Memory-mapped (pockets, PoseLibrary); arrays are views into the file."""
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    if bytes(mm[:8]) != MAGIC:
        raise ValueError(f"{path}: not a packed pose library")
    n_pk, n_pa, n_p, n_a = (int(x) for x in np.frombuffer(mm[8:40], dtype="<u8"))
    off = 40
    out = []
    for dt, count in (("<i8", n_pk + 1), ("<f8", n_pa * 3), ("<i4", n_pa), ("<i4", n_pa), ("<i8", n_p + 1),
                      ("<i4", n_p), ("<i8", n_p), ("<i8", n_p), ("<f8", n_a * 3), ("<i4", n_a), ("<i4", n_a)):
        off = (off + _ALIGN - 1) // _ALIGN * _ALIGN
        nbytes = np.dtype(dt).itemsize * count
        out.append(np.frombuffer(mm[off:off + nbytes], dtype=dt))
        off += nbytes
    p_off, p_xyz, p_el, p_ro, a_off, tgt, comp, pid, xyz, el, ro = out
    pockets = [Pocket(p_xyz.reshape(-1, 3)[p_off[i]:p_off[i + 1]], p_el[p_off[i]:p_off[i + 1]],
                      p_ro[p_off[i]:p_off[i + 1]], f"pocket{i}") for i in range(n_pk)]
    lib = PoseLibrary(xyz.reshape(-1, 3), el, ro, a_off, tgt, comp, pid)
    return pockets, lib


class StreamingLoader:
    """Double-buffered pinned staging of library batches onto one device.

    ``for s, e, batch, compound, pose_id in loader.batches():`` yields device
    views whose H2D copy was issued on a side stream and is ordered before
    use on the current stream (event wait); the copy of the next batch
    overlaps.  Same protocol as screen.DeviceLibrary.batches."""

    @property
    def n_poses(self):
        return self.lib.n_poses

    def __init__(self, lib: PoseLibrary, pockets, batch_size: int, device=None, index_base=0):
        import torch

        from . import engine as E
        self.torch, self.E = torch, E
        self.lib, self.B = lib, int(batch_size)
        self.index_base = int(index_base)
        self.device = E._require_cuda(device)
        P = lib.n_poses
        self.bounds = [(s, min(P, s + self.B)) for s in range(0, P, self.B)]
        max_atoms = max((int(lib.atom_off[e] - lib.atom_off[s]) for s, e in self.bounds), default=1)
        pk_off = np.concatenate([[0], np.cumsum([len(p.xyz) for p in pockets])]).astype(np.int64)
        dev = self.device
        self.pocket = dict(
            pocket_xyz=torch.from_numpy(np.ascontiguousarray(np.concatenate([p.xyz for p in pockets]))).to(dev),
            pocket_elem=torch.from_numpy(np.concatenate([p.elem for p in pockets]).astype(np.int32)).to(dev),
            pocket_role=torch.from_numpy(np.concatenate([p.role for p in pockets]).astype(np.int32)).to(dev),
            pocket_off=torch.from_numpy(pk_off).to(dev))
        psz = np.diff(pk_off)
        self.max_pose_atoms = int((np.diff(lib.atom_off) + psz[lib.target]).max()) if P else 1
        self.h2d_bytes = 0
        # two pinned host slots + two device slots
        self.slots = []
        for _ in range(2):
            h = dict(xyz=torch.empty((max_atoms, 3), dtype=torch.float64).pin_memory(),
                     elem=torch.empty(max_atoms, dtype=torch.int32).pin_memory(),
                     role=torch.empty(max_atoms, dtype=torch.int32).pin_memory(),
                     off=torch.empty(self.B + 1, dtype=torch.int64).pin_memory(),
                     tgt=torch.empty(self.B, dtype=torch.int32).pin_memory(),
                     comp=torch.empty(self.B, dtype=torch.int64).pin_memory(),
                     pid=torch.empty(self.B, dtype=torch.int64).pin_memory())
            d = {k: torch.empty_like(v, device=dev) for k, v in h.items()}
            self.slots.append((h, d, torch.cuda.Event()))
        self.copy_stream = torch.cuda.Stream(device=dev)

    def _stage(self, i):
        torch = self.torch
        s, e = self.bounds[i]
        h, d, ev = self.slots[i % 2]
        a, b = int(self.lib.atom_off[s]), int(self.lib.atom_off[e])
        n = b - a
        ev.synchronize()          # the slot's previous H2D copy has drained the pinned buffer
        h["xyz"][:n].numpy()[:] = self.lib.xyz[a:b]                 # memmap -> pinned
        h["elem"][:n].numpy()[:] = self.lib.elem[a:b]
        h["role"][:n].numpy()[:] = self.lib.role[a:b]
        h["off"][: e - s + 1].numpy()[:] = self.lib.atom_off[s:e + 1] - a
        h["tgt"][: e - s].numpy()[:] = self.lib.target[s:e]
        h["comp"][: e - s].numpy()[:] = self.lib.compound[s:e]
        h["pid"][: e - s].numpy()[:] = self.lib.pose_id[s:e]
        with torch.cuda.stream(self.copy_stream):
            for k, cnt in (("xyz", n), ("elem", n), ("role", n), ("off", e - s + 1), ("tgt", e - s),
                           ("comp", e - s), ("pid", e - s)):
                d[k][:cnt].copy_(h[k][:cnt], non_blocking=True)
            ev.record(self.copy_stream)
        self.h2d_bytes += n * 32 + (e - s + 1) * 8 + (e - s) * 20
        return s, e, d, ev

    def batches(self, batch_size=None):
        if batch_size is not None and int(batch_size) != self.B:
            raise ValueError(f"StreamingLoader was built for batch {self.B}, asked for {batch_size}")
        torch = self.torch
        if not self.bounds:
            return
        pending = self._stage(0)
        for i in range(len(self.bounds)):
            s, e, d, ev = pending
            torch.cuda.current_stream().wait_event(ev)
            batch = self.E.PoseBatch(
                d["xyz"], d["elem"], d["role"], d["off"][: e - s + 1], self.max_pose_atoms,
                self.pocket["pocket_xyz"], self.pocket["pocket_elem"], self.pocket["pocket_role"],
                self.pocket["pocket_off"], d["tgt"][: e - s])
            if i + 1 < len(self.bounds):
                # the slot of batch i+1 was last read by batch i-1, which the
                # caller's stream has consumed before asking for batch i
                self.copy_stream.wait_stream(torch.cuda.current_stream())
                pending = self._stage(i + 1)
            yield s, e, batch, d["comp"][: e - s], d["pid"][: e - s]
