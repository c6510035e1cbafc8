"""Synthetic docked-pose libraries for pocket screens (BASELINE configs 1,4,5).

The distribution is the reference's ``generate_complex`` (complexes.py:107-119)
restated for screening: a *pocket* (protein atoms ~U[-b/2, b/2)^3, elements
~U{0..c-1}, role PROTEIN) is shared by every pose of a target, and each
*compound* has a ligand (size ~U{lo..hi}, elements ~U{0..c-1}) docked in
several *poses* (centre ~U[-b/8, b/8)^3, atoms clip(centre + N(0, 1.8^2),
+-b/2), role LIGAND).  Pose p of a screen is the complex
``vstack([pocket, ligand pose p])`` -- exactly what the reference scores.
All draws are vectorised numpy with explicit seeds.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PROTEIN, LIGAND = 0, 1


@dataclass
class Pocket:
    xyz: np.ndarray      # [n,3] float64
    elem: np.ndarray     # [n] int32
    role: np.ndarray     # [n] int32 (all PROTEIN)
    name: str = "pocket"


@dataclass
class PoseLibrary:
    xyz: np.ndarray          # [A,3] float64 ligand atoms of all poses
    elem: np.ndarray         # [A] int32
    role: np.ndarray         # [A] int32 (all LIGAND)
    atom_off: np.ndarray     # [P+1] int64
    target: np.ndarray       # [P] int32 pocket index
    compound: np.ndarray     # [P] int64 compound id
    pose_id: np.ndarray      # [P] int64 pose id within compound

    @property
    def n_poses(self):
        return len(self.atom_off) - 1

    def slice(self, s, e) -> "PoseLibrary":
        a, b = self.atom_off[s], self.atom_off[e]
        return PoseLibrary(self.xyz[a:b], self.elem[a:b], self.role[a:b], self.atom_off[s:e + 1] - a,
                           self.target[s:e], self.compound[s:e], self.pose_id[s:e])


def make_pocket(n_atoms=1000, seed=0, box_size=16.0, c_elem=4, name="pocket") -> Pocket:
    rng = np.random.default_rng(seed)
    half = box_size / 2.0
    xyz = rng.uniform(-half, half, size=(n_atoms, 3))
    elem = rng.integers(0, c_elem, size=n_atoms).astype(np.int32)
    return Pocket(xyz, elem, np.full(n_atoms, PROTEIN, dtype=np.int32), name)


def make_poses(n_compounds, poses_per_compound=10, seed=1, ligand_atoms=(16, 64), box_size=16.0,
               c_elem=4, target=0, compound_base=0) -> PoseLibrary:
    """Ligand poses for ``n_compounds`` compounds x ``poses_per_compound``."""
    rng = np.random.default_rng(seed)
    half = box_size / 2.0
    lo, hi = ligand_atoms
    n_lig = rng.integers(lo, hi + 1, size=n_compounds)
    lig_elem = rng.integers(0, c_elem, size=int(n_lig.sum())).astype(np.int32)
    lig_off = np.concatenate([[0], np.cumsum(n_lig)])
    per_pose = np.repeat(n_lig, poses_per_compound)
    P = len(per_pose)
    atom_off = np.concatenate([[0], np.cumsum(per_pose)]).astype(np.int64)
    A = int(atom_off[-1])
    centres = rng.uniform(-half / 4, half / 4, size=(P, 3))
    pose_of_atom = np.repeat(np.arange(P), per_pose)
    xyz = np.clip(centres[pose_of_atom] + rng.normal(0.0, 1.8, size=(A, 3)), -half, half)
    # each pose of a compound repeats the compound's element list
    comp_of_pose = np.repeat(np.arange(n_compounds), poses_per_compound)
    within = np.arange(A) - atom_off[pose_of_atom]
    elem = lig_elem[lig_off[comp_of_pose[pose_of_atom]] + within]
    return PoseLibrary(xyz=xyz, elem=elem.astype(np.int32), role=np.full(A, LIGAND, dtype=np.int32),
                       atom_off=atom_off, target=np.full(P, target, dtype=np.int32),
                       compound=(comp_of_pose + compound_base).astype(np.int64),
                       pose_id=np.tile(np.arange(poses_per_compound), n_compounds).astype(np.int64))


def concat(libs) -> PoseLibrary:
    offs, total = [], 0
    for lib in libs:
        offs.append(lib.atom_off[:-1] + total)
        total += int(lib.atom_off[-1])
    return PoseLibrary(np.concatenate([l.xyz for l in libs]), np.concatenate([l.elem for l in libs]),
                       np.concatenate([l.role for l in libs]),
                       np.concatenate(offs + [np.array([total], dtype=np.int64)]).astype(np.int64),
                       np.concatenate([l.target for l in libs]), np.concatenate([l.compound for l in libs]),
                       np.concatenate([l.pose_id for l in libs]))


def complex_arrays(pocket: Pocket, lib: PoseLibrary, p: int):
    """Full complex (positions, elements, roles) of pose p: vstack([pocket, ligand])."""
    a, b = lib.atom_off[p], lib.atom_off[p + 1]
    return (np.vstack([pocket.xyz, lib.xyz[a:b]]), np.concatenate([pocket.elem, lib.elem[a:b]]).astype(np.int64),
            np.concatenate([pocket.role, lib.role[a:b]]).astype(np.int64))


# Target pockets of BASELINE config 5.  The paper gives no atom counts, only
# "Mpro sites are large protein pockets and the spike targets are much
# smaller"; sizes below are the stated proposal.
FOUR_TARGETS = (("protease1", 1000), ("protease2", 900), ("spike1", 450), ("spike2", 350))
