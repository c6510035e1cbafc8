"""Drop-in featurizer API of ``fusionscreen.complexes`` on the B200 path.

Same names, argument meaning and errors as the reference
(/root/reference/pkg/src/fusionscreen/complexes.py); ``voxelize`` and
``build_graph`` run the CUDA kernels of libfusionb200 (no CPU fallback).
Batched forms (``voxelize_batch``, ``build_graph_batch``) featurize whole
libraries in one launch each -- the screening path never loops per pose.

Out of scope here (data preparation, not the scoring path): rotate_augment,
quintile_split, manifest IO.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, field

import numpy as np

PROTEIN, LIGAND = 0, 1                      # complexes.py:26
THRESHOLD_RANGE = (1.2, 5.9)                # complexes.py:207
CONTACT_WEIGHT, DISTANCE_WEIGHT, CONTACT_CUTOFF = 0.2, 0.5, 4.0   # complexes.py:29-31


@dataclass(frozen=True)
class GenParams:
    """Generation knobs (complexes.py:51-68)."""

    box_size: float = 16.0
    c_elem: int = 4
    n_protein: tuple = (20, 60)
    n_ligand: tuple = (5, 20)
    noise_sigma: float = 0.25

    def validate(self):
        if self.box_size <= 0:
            raise ValueError("box_size must be positive")
        if self.c_elem < 1:
            raise ValueError("c_elem must be >= 1")
        for lo, hi in (self.n_protein, self.n_ligand):
            if lo < 1 or hi < lo:
                raise ValueError("atom count ranges must satisfy 1 <= lo <= hi")


@dataclass
class SyntheticComplex:
    """One pose (complexes.py:71-88): positions [n,3] A, elements, roles."""

    complex_id: str
    positions: np.ndarray
    elements: np.ndarray
    roles: np.ndarray
    label_pk: float
    meta: dict = field(default_factory=dict)

    @property
    def n_atoms(self) -> int:
        return len(self.positions)

    def protein_mask(self):
        return self.roles == PROTEIN

    def ligand_mask(self):
        return self.roles == LIGAND


def planted_label(positions, roles) -> float:
    """Noise-free planted affinity, clamped to [0, 12] (complexes.py:91-99).
    Host-side label synthesis (not on the scoring path)."""
    from scipy.spatial.distance import cdist
    d = cdist(positions[roles == LIGAND], positions[roles == PROTEIN])
    f = CONTACT_WEIGHT * int((d < CONTACT_CUTOFF).sum()) - DISTANCE_WEIGHT * float(d.min(axis=1).mean())
    return float(np.clip(f, 0.0, 12.0))


def generate_complex(seed: int, gen_params: GenParams = GenParams()) -> SyntheticComplex:
    """Seeded synthetic complex with the reference's distribution and draw
    order (complexes.py:102-130): protein ~U[-b/2,b/2)^3, ligand =
    clip(centre + N(0,1.8^2)), centre ~U[-b/8,b/8)^3, elements ~U{0..c-1}."""
    gp = gen_params
    gp.validate()
    rng = np.random.default_rng(seed)
    half = gp.box_size / 2.0
    n_prot = int(rng.integers(gp.n_protein[0], gp.n_protein[1] + 1))
    n_lig = int(rng.integers(gp.n_ligand[0], gp.n_ligand[1] + 1))
    prot = rng.uniform(-half, half, size=(n_prot, 3))
    centre = rng.uniform(-half / 4, half / 4, size=3)
    lig = np.clip(centre + rng.normal(0.0, 1.8, size=(n_lig, 3)), -half, half)
    positions = np.vstack([prot, lig])
    roles = np.concatenate([np.full(n_prot, PROTEIN, dtype=np.int64), np.full(n_lig, LIGAND, dtype=np.int64)])
    elements = rng.integers(0, gp.c_elem, size=n_prot + n_lig)
    label = planted_label(positions, roles)
    if gp.noise_sigma > 0:
        label += float(rng.normal(0.0, gp.noise_sigma))
    return SyntheticComplex(f"cpx-{seed:08d}", positions, elements, roles, label,
                            {"seed": int(seed), "gen_params": asdict(gp)})


def generate_dataset(count: int, seed: int, gen_params: GenParams = GenParams()):
    base = np.random.default_rng(seed).integers(0, 2 ** 31 - 1)     # complexes.py:133-136
    return [generate_complex(int(base) + i, gen_params) for i in range(count)]


@dataclass(frozen=True)
class GridConfig:
    extent: int = 16
    c_elem: int = 4
    box_size: float = 16.0

    def validate(self):
        if self.extent < 8:
            raise ValueError(f"grid extent must be >= 8, got {self.extent}")

    @property
    def channels(self) -> int:
        return 2 * self.c_elem


@dataclass
class VoxelGrid:
    occupancy: np.ndarray   # [2*c_elem, G, G, G]

    @property
    def channels(self) -> int:
        return self.occupancy.shape[0]

    @property
    def extent(self) -> int:
        return self.occupancy.shape[1]


@dataclass
class ComplexGraph:
    node_features: np.ndarray
    covalent_edges: np.ndarray
    noncovalent_edges: np.ndarray
    covalent_dists: np.ndarray
    noncovalent_dists: np.ndarray

    @property
    def n_nodes(self) -> int:
        return len(self.node_features)


# ---------------------------------------------------------------------------
# GPU featurization
# ---------------------------------------------------------------------------

def _engine():
    from . import engine
    return engine


def _raise_item_errors(err, what):
    from . import _native as N
    err = np.asarray(err)
    bad = np.flatnonzero(err)
    if len(bad):
        e = int(err[bad[0]])
        if e & N.FS_ERR_ROLE:
            raise IndexError(f"{what}: role outside {{PROTEIN, LIGAND}} in complex {bad[0]}")
        if e & (N.FS_ERR_NAN | N.FS_ERR_NONFINITE):
            raise ValueError(f"{what}: non-finite coordinates in complex {bad[0]}")
        if e & N.FS_ERR_TOO_LARGE:
            raise ValueError(f"{what}: complex {bad[0]} exceeds {N.FS_MAX_POSE_ATOMS} atoms")
        raise RuntimeError(f"{what}: device error flags {e} for complex {bad[0]}")


def voxelize_batch(complexes, grid: GridConfig = GridConfig()) -> np.ndarray:
    """Voxel grids of many complexes in one launch: float64 [P, C, G, G, G]."""
    grid.validate()
    E = _engine()
    b = E.batch_from_complexes(complexes)
    occ, err = E.voxelize(b, grid.extent, grid.c_elem, grid.box_size)
    _raise_item_errors(err.cpu().numpy(), "voxelize")
    return occ.cpu().numpy()


def voxelize(c: SyntheticComplex, grid: GridConfig = GridConfig()) -> VoxelGrid:
    """complexes.voxelize (complexes.py:171-184) on the GPU, bit-exact."""
    return VoxelGrid(voxelize_batch([c], grid)[0])


def _check_thresholds(*ts):
    lo, hi = THRESHOLD_RANGE
    for t in ts:
        if not lo <= t <= hi:
            raise ValueError(f"threshold {t} outside searched range [{lo}, {hi}]")


def build_graph_batch(complexes, cov_thresh: float = 2.24, noncov_thresh: float = 5.22,
                      c_elem: int = 4, box_size: float = 16.0) -> list:
    """build_graph for many complexes: one count + one fill launch in total.

    Edges are emitted in canonical (i, j)-lexsorted order (the reference emits
    kd-tree traversal order; the edge *sets* and distances are bit-identical)."""
    _check_thresholds(cov_thresh, noncov_thresh)
    E = _engine()
    b = E.batch_from_complexes(complexes)
    g = E.radius_graph(b, cov_thresh, noncov_thresh, with_dists=True)
    _raise_item_errors(g.err.cpu().numpy(), "build_graph")
    feats = E.node_features(b, g.node_off, c_elem, box_size).cpu().numpy()
    ce, cd, coff = E.edge_lists(g, "cov")
    ne, nd, noff = E.edge_lists(g, "ncov")
    ce, cd, coff = ce.cpu().numpy(), cd.cpu().numpy(), coff.cpu().numpy()
    ne, nd, noff = ne.cpu().numpy(), nd.cpu().numpy(), noff.cpu().numpy()
    node_off = g.node_off.cpu().numpy()
    out = []
    for p in range(len(complexes)):
        out.append(ComplexGraph(
            node_features=feats[node_off[p]:node_off[p + 1]],
            covalent_edges=ce[coff[p]:coff[p + 1]].reshape(-1, 2),
            noncovalent_edges=ne[noff[p]:noff[p + 1]].reshape(-1, 2),
            covalent_dists=cd[coff[p]:coff[p + 1]],
            noncovalent_dists=nd[noff[p]:noff[p + 1]]))
    return out


def build_graph(c: SyntheticComplex, cov_thresh: float = 2.24, noncov_thresh: float = 5.22,
                c_elem: int = 4, box_size: float = 16.0) -> ComplexGraph:
    """complexes.build_graph (complexes.py:223-254) on the GPU."""
    return build_graph_batch([c], cov_thresh, noncov_thresh, c_elem, box_size)[0]
