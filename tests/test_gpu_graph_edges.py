"""Bit-exact edge lists of the radius graph the SCORING path runs.

fs_scoring_graph runs the graph kernels exactly as fs_score_poses
(graph_csr_kernel) and fs_score_poses_cached (graph_fact_kernel) launch them
and lists every directed CSR entry the SG-CNN reads; these tests compare those
entries and their float64 distances bitwise with the reference's build_graph
rule (complexes.py:237-246), through the committed reference goldens and the
pinned C oracle (oracle/radius_graph.c) at config-2 scale.
"""

import numpy as np
import pytest
import torch

from oracle import radius_c
from paper_2104_04547_b200 import engine as E
from paper_2104_04547_b200 import synth
from tests._cfg import load

pytestmark = pytest.mark.gpu

TC, TN = 2.24, 5.22


def _gpu_entries(batch, max_edges, factored=False, max_pocket=0):
    out = E.scoring_graph_entries(batch, TC, TN, max_edges, factored, max_pocket)
    torch.cuda.synchronize()
    res = {"err": out["err"].cpu().numpy()}
    for t in ("cov", "ncov"):
        n = out[f"n_{t}"].to(torch.int64)
        mask = torch.arange(max_edges, device=n.device)[None, :] < n[:, None]
        res[f"n_{t}"] = n.cpu().numpy()
        res[f"ent_{t}"] = out[f"ent_{t}"][mask].cpu().numpy().astype(np.int64)
        res[f"d_{t}"] = out[f"d_{t}"][mask].cpu().numpy()
    return res


def _keys(pose, i, j):
    return (pose.astype(np.int64) << 26) | (i.astype(np.int64) << 13) | j.astype(np.int64)


def _compare(got, want_edges, want_d, want_off, t, poses=None):
    """Directed GPU entries == both orientations of the oracle's i<j edges;
    distances bitwise.  `poses` restricts the check to a subset."""
    P = len(want_off) - 1
    n = got[f"n_{t}"]
    pose_of = np.repeat(np.arange(P), n)
    ent, d = got[f"ent_{t}"], got[f"d_{t}"]
    wp = np.repeat(np.arange(P), np.diff(want_off))
    wi, wj = want_edges[:, 0], want_edges[:, 1]
    if poses is not None:
        keep = np.isin(pose_of, poses)
        pose_of, ent, d = pose_of[keep], ent[keep], d[keep]
        wk = np.isin(wp, poses)
        wp, wi, wj, want_d = wp[wk], wi[wk], wj[wk], want_d[wk]
    gk = _keys(pose_of, ent[:, 0], ent[:, 1])
    wk = np.concatenate([_keys(wp, wi, wj), _keys(wp, wj, wi)])
    wd = np.concatenate([want_d, want_d])
    og, ow = np.argsort(gk, kind="stable"), np.argsort(wk, kind="stable")
    assert len(gk) == len(wk), (t, len(gk), len(wk))
    assert np.array_equal(gk[og], wk[ow]), t
    assert np.array_equal(d[og].view(np.uint64), wd[ow].view(np.uint64)), t   # float64 bitwise


def _complex_batch(pos, roles, elems, off, max_pose_atoms=None):
    b = E.batch_from_arrays(pos, elems, roles, off)
    if max_pose_atoms is not None:
        b.max_pose_atoms = max_pose_atoms
    return b


def _oracle(pos, roles, off):
    return radius_c.radius_pairs_batch(pos, roles, off, TC, TN)


@pytest.mark.parametrize("name", ["featurize_golden.npz", "graph_edge_golden.npz"])
def test_scoring_graph_matches_reference_goldens(name):
    """Every golden complex (threshold-exact and +-1 ulp pairs, ligand > 64
    atoms, swapped role sizes, |coords| >= 1024 A, > 96 covalent candidates per
    row, coincident atoms, single-atom and single-role poses) against the
    reference's own build_graph output."""
    from oracle import fusion_oracle as orc
    z = load(name)
    off = z["atom_off"]
    got = _gpu_entries(_complex_batch(z["positions"], z["roles"], z["elements"], off), 65536)
    assert not got["err"].any()
    for t in ("cov", "ncov"):
        edges, dists, eoff = [], [], [0]
        for p in range(len(off) - 1):
            s, e = z[f"{t}_off"][p], z[f"{t}_off"][p + 1]
            ce, cd = orc.canonical_edges(z[f"{t}_edges"][s:e], z[f"{t}_dists"][s:e])
            edges.append(ce)
            dists.append(cd)
            eoff.append(eoff[-1] + len(ce))
        _compare(got, np.concatenate(edges), np.concatenate(dists), np.array(eoff), t)


def _screen_arrays(n_comp, seed, pocket_atoms=1000, ligand_atoms=(16, 64), shift=0.0):
    pk = synth.make_pocket(pocket_atoms, seed=seed)
    lib = synth.make_poses(n_comp, 10, seed=seed + 1, ligand_atoms=ligand_atoms)
    pk.xyz = pk.xyz + shift
    lib.xyz = lib.xyz + shift
    return pk, lib


def _full_arrays(pk, lib):
    """Concatenated complexes vstack([pocket, ligand]) for the oracle."""
    P = lib.n_poses
    lig = np.diff(lib.atom_off)
    off = np.concatenate([[0], np.cumsum(lig + len(pk.xyz))]).astype(np.int64)
    pos = np.empty((off[-1], 3))
    roles = np.empty(off[-1], dtype=np.int64)
    for p in range(P):
        a, b = off[p], off[p + 1]
        pos[a:a + len(pk.xyz)] = pk.xyz
        pos[a + len(pk.xyz):b] = lib.xyz[lib.atom_off[p]:lib.atom_off[p + 1]]
        roles[a:a + len(pk.xyz)] = 0
        roles[a + len(pk.xyz):b] = 1
    return pos, roles, off


def _pocket_batch(pk, lib):
    return E.batch_from_arrays(lib.xyz, lib.elem, lib.role, lib.atom_off,
                               pocket=(pk.xyz, pk.elem, pk.role, np.array([0, len(pk.xyz)])),
                               pose_target=lib.target)


def test_scoring_graph_config2_sample_bitwise():
    """Config 2 sample: 10,240 BASELINE-shape poses (1,000-atom pockets,
    ligands U{16..64}, 10 pocket seeds), every directed entry and distance of
    the scoring-path graph bitwise equal to the C oracle."""
    total = 0
    for chunk in range(10):
        pk, lib = _screen_arrays(103, seed=100 + 7 * chunk)
        lib = lib.slice(0, 1024)
        got = _gpu_entries(_pocket_batch(pk, lib), 32768)
        assert not got["err"].any()
        pos, roles, off = _full_arrays(pk, lib)
        ce, cd, coff, ne, nd, noff = _oracle(pos, roles, off)
        _compare(got, ce, cd, coff, "cov")
        _compare(got, ne, nd, noff, "ncov")
        total += lib.n_poses
    assert total == 10240


def test_scoring_graph_far_coordinates_and_big_ligands():
    """|coords| >= 1024 A (fp32 prefilter off: every pair decided in float64)
    and ligands of 65-200 atoms (non-covalent bitmask path off)."""
    for shift, lig in ((2048.0, (16, 64)), (-1500.0, (65, 200)), (0.0, (65, 200))):
        pk, lib = _screen_arrays(26, seed=31, pocket_atoms=700, ligand_atoms=lig, shift=shift)
        got = _gpu_entries(_pocket_batch(pk, lib), 65536)      # 200-atom ligands: > 32k directed entries
        assert not got["err"].any()
        pos, roles, off = _full_arrays(pk, lib)
        ce, cd, coff, ne, nd, noff = _oracle(pos, roles, off)
        _compare(got, ce, cd, coff, "cov")
        _compare(got, ne, nd, noff, "ncov")


def _ulp_poses(n_poses, seed):
    """Poses whose ligand atoms sit at exactly t, t-1ulp, t+1ulp from a pocket
    or ligand atom in random directions (the in-band float64 path)."""
    rng = np.random.default_rng(seed)
    pk, lib = _screen_arrays(n_poses // 10 + 1, seed=seed, pocket_atoms=600)
    lib = lib.slice(0, n_poses)
    xyz = lib.xyz.copy()
    for p in range(n_poses):
        a, b = lib.atom_off[p], lib.atom_off[p + 1]
        for k in range(a + 1, b):
            u = rng.normal(size=3)
            u /= np.linalg.norm(u)
            t = TN if k % 2 else TC
            d = (np.nextafter(t, 0), t, np.nextafter(t, 10))[k % 3]
            anchor = pk.xyz[rng.integers(len(pk.xyz))] if k % 2 else xyz[k - 1]
            xyz[k] = anchor + d * u
    lib.xyz = xyz
    return pk, lib


def test_scoring_graph_threshold_ulp_cases():
    pk, lib = _ulp_poses(300, seed=5)
    got = _gpu_entries(_pocket_batch(pk, lib), 32768)
    assert not got["err"].any()
    pos, roles, off = _full_arrays(pk, lib)
    ce, cd, coff, ne, nd, noff = _oracle(pos, roles, off)
    _compare(got, ce, cd, coff, "cov")
    _compare(got, ne, nd, noff, "ncov")


def test_scoring_graph_compressed_pockets():
    """Pockets squeezed into a small box: crowded cells (> 64 atoms per
    stencil column) and > 96 covalent candidates per row (the re-test path)."""
    rng = np.random.default_rng(9)
    pk, lib = _screen_arrays(4, seed=77, pocket_atoms=500)
    pk.xyz = rng.uniform(-2.6, 2.6, size=(500, 3))
    got = _gpu_entries(_pocket_batch(pk, lib), 65536)
    assert not got["err"].any()
    pos, roles, off = _full_arrays(pk, lib)
    ce, cd, coff, ne, nd, noff = _oracle(pos, roles, off)
    assert (np.diff(coff) > 20000).all()
    _compare(got, ce, cd, coff, "cov")
    _compare(got, ne, nd, noff, "ncov")


@pytest.mark.parametrize("pocket_atoms,lig", [(1000, (16, 64)), (450, (16, 128)), (350, (100, 128))])
def test_factored_scoring_graph_bitwise(pocket_atoms, lig):
    """fs_score_poses_cached's graph: ligand-ligand covalent and ligand-pocket
    non-covalent entries (pocket-pocket edges come from the pocket cache,
    built by graph_csr_kernel and covered above), bitwise."""
    pk, lib = _screen_arrays(52, seed=200 + pocket_atoms, pocket_atoms=pocket_atoms, ligand_atoms=lig)
    got = _gpu_entries(_pocket_batch(pk, lib), 32768, factored=True, max_pocket=pocket_atoms)
    assert not got["err"].any()
    pos, roles, off = _full_arrays(pk, lib)
    ce, cd, coff, ne, nd, noff = _oracle(pos, roles, off)
    lig_only = (ce[:, 0] >= pocket_atoms)        # i<j, so both ends are ligand atoms
    cp = np.repeat(np.arange(lib.n_poses), np.diff(coff))
    coff2 = np.concatenate([[0], np.cumsum(np.bincount(cp[lig_only], minlength=lib.n_poses))])
    _compare(got, ce[lig_only], cd[lig_only], coff2, "cov")
    _compare(got, ne, nd, noff, "ncov")


@pytest.mark.parametrize("shift", [0.0, 2048.0])
def test_factored_scoring_graph_threshold_ulp_and_far_cases(shift):
    """The factored graph's exact float64 settle: ligand atoms at t, t - 1 ulp
    and t + 1 ulp from pocket / ligand atoms (the fp32 band), and the same
    poses moved to |coords| >= 1024 A (prefilter off), bitwise."""
    pk, lib = _ulp_poses(200, seed=11)
    pk.xyz = pk.xyz + shift
    lib.xyz = lib.xyz + shift
    got = _gpu_entries(_pocket_batch(pk, lib), 32768, factored=True, max_pocket=len(pk.xyz))
    assert not got["err"].any()
    pos, roles, off = _full_arrays(pk, lib)
    ce, cd, coff, ne, nd, noff = _oracle(pos, roles, off)
    lig_only = (ce[:, 0] >= len(pk.xyz))
    cp = np.repeat(np.arange(lib.n_poses), np.diff(coff))
    coff2 = np.concatenate([[0], np.cumsum(np.bincount(cp[lig_only], minlength=lib.n_poses))])
    _compare(got, ce[lig_only], cd[lig_only], coff2, "cov")
    _compare(got, ne, nd, noff, "ncov")


def test_factored_graph_flags_oversize_ligands():
    pk, lib = _screen_arrays(3, seed=3, pocket_atoms=300, ligand_atoms=(129, 140))
    got = _gpu_entries(_pocket_batch(pk, lib), 32768, factored=True, max_pocket=300)
    from paper_2104_04547_b200 import _native as N
    assert np.all(got["err"] & N.FS_ERR_NOT_FACTORED)


def test_oversize_pose_is_flagged_without_touching_others():
    """A pose above the caller's max_pose_atoms bound gets FS_ERR_TOO_LARGE and
    writes nothing outside its own rows; the other poses' graphs are intact
    (node rows are clamped to the bound)."""
    from paper_2104_04547_b200 import _native as N
    pk, lib = _screen_arrays(1, seed=8, pocket_atoms=200)
    pos, roles, off = _full_arrays(pk, lib)
    # make pose 3 oversize: append 150 extra ligand atoms to it
    extra = np.random.default_rng(0).uniform(-8, 8, (150, 3))
    a, b = off[3], off[4]
    pos = np.vstack([pos[:b], extra, pos[b:]])
    roles = np.concatenate([roles[:b], np.ones(150, dtype=np.int64), roles[b:]])
    off = off.copy()
    off[4:] += 150
    elems = np.zeros(len(roles), dtype=np.int64)
    bound = int(np.delete(np.diff(off), 3).max())
    got = _gpu_entries(_complex_batch(pos, roles, elems, off, max_pose_atoms=bound), 32768)
    assert got["err"][3] & N.FS_ERR_TOO_LARGE
    assert not np.delete(got["err"], 3).any()
    ce, cd, coff, ne, nd, noff = _oracle(pos, roles, off)
    others = [p for p in range(len(off) - 1) if p != 3]
    _compare(got, ce, cd, coff, "cov", poses=others)
    _compare(got, ne, nd, noff, "ncov", poses=others)
