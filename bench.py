"""Throughput bench of the B200 Coherent-Fusion pose-scoring path.

Headline workload (BASELINE.json configs[3], "config 4"): a screen of
1,000,000 synthetic docked poses (100,000 compounds x 10 poses) against one
1,000-atom pocket; ligands U{16..64} atoms; random-init weights
FusionModel(seed=0).  The screen is fixed and sharded over the N ranks
(compound-aligned contiguous shards, strong scaling); each rank scores its
shard in exactly K steps.  A *step* is one fused pass of the hot path --
featurize (voxel splat + exact radius graph) + 3D-CNN + SG-CNN + fusion +
running device top-k and per-compound best pose -- over one batch of the
rank's poses.  The only collective is the final NCCL all-gather of the
per-rank top-k (merged on device), inside the timed region.
(``--scaling weak``: K batches of --batch poses per rank instead.)

At N=1 rank 0 also reports, beside the headline line:
  parity       -- BASELINE config 1 (1,024 poses, batch 32) scored in fp32,
                  mixed and bf16 against the CPU oracle, per-pose errors and
                  top-k equality; the oracle run is also the CPU baseline
                  (all host cores, 1 BLAS thread each)
  plugin       -- end-to-end throughput through the reference-facing API:
                  ModelScorer(list[PoseRecord]) with raw complexes, and
                  predict_batch with featurized items, host buffers in
                  and scores out
  configs      -- BASELINE configs 2 (featurizer only), 3 (each branch
                  alone, fp32 and bf16) and 5 (4-target screen, variable
                  ligand sizes)
  roofline     -- per-kernel fractions from a serial (non-overlapped) pass

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precision bf16|mixed|fp32]
    python bench.py --impl reference ...   # CPU reference arm (oracle port)
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "docked poses scored/sec (8×B200, device-timed) vs CPU ref; roofline fraction"
POCKET_ATOMS = 1000
LIGAND_ATOMS = (16, 64)
POSES_PER_COMPOUND = 10
SCREEN_COMPOUNDS = 100_000            # config 4: 1M poses
CHUNK_COMPOUNDS = 1000                # library generation unit (independent of N)
TOPK = 100
WORKLOAD = ("config4: Coherent Fusion screen of 1,000,000 poses vs one 1000-atom pocket, ligands U{16..64} atoms, "
            "10 poses/compound, sharded over the ranks; featurize+3D-CNN+SG-CNN+fusion+top-k per step")

# algorithmic work per pose: FLOP(N,Ec,En)
VOXEL_FLOP = 659_570_816
CONV_FLOP = {"conv1": 2 * 131_072_000, "conv2": 2 * 113_246_208, "conv3": 2 * 28_311_552,
             "conv4": 2 * 56_623_104}
DENSE_FLOP = 2 * (4096 * 128 + 128 * 64)
# fraction of CONV_FLOP the tensor cores actually issue: the kernels skip the
# all-zero "same"-padding depth planes (umma_conv.cu issuer), i.e. the
# R(R+1) of G*KS (input plane, output plane) pairs that read only padding
CONV_GKS = {"conv1": (16, 5), "conv2": (16, 3), "conv3": (8, 3), "conv4": (8, 3)}
CONV_ISSUED = {k: 1.0 - (ks // 2) * (ks // 2 + 1) / (g * ks) for k, (g, ks) in CONV_GKS.items()}


def graph_flop(n, ec, en):
    return 85_248 * n + 28_984 + 48 * (6 * ec + 3 * en)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.mark_at = 0

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "20",
                 "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.mark_at = 0
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def ready(self, timeout=5.0):
        """Wait for the sampler's first line (nvidia-smi starts slowly), then
        mark where the timed region's samples begin."""
        t0 = time.perf_counter()
        while self.proc and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)
        self.mark_at = len(self.lines)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        lines = self.lines[self.mark_at:] or self.lines[-1:]
        for ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# synthetic libraries (deterministic, independent of the rank count)
# ---------------------------------------------------------------------------
def screen_library(c0, c1, seed=1, ligand_atoms=LIGAND_ATOMS, target=0):
    """Compounds [c0, c1) of the global screen: generated chunk by chunk
    (chunk j from seed + j), so every rank count sees the same library."""
    from paper_2104_04547_b200 import synth
    parts = []
    for j in range(c0 // CHUNK_COMPOUNDS, (c1 + CHUNK_COMPOUNDS - 1) // CHUNK_COMPOUNDS):
        ch = synth.make_poses(CHUNK_COMPOUNDS, POSES_PER_COMPOUND, seed=seed + j, ligand_atoms=ligand_atoms,
                              target=target, compound_base=j * CHUNK_COMPOUNDS)
        a = max(c0, j * CHUNK_COMPOUNDS) - j * CHUNK_COMPOUNDS
        b = min(c1, (j + 1) * CHUNK_COMPOUNDS) - j * CHUNK_COMPOUNDS
        parts.append(ch.slice(a * POSES_PER_COMPOUND, b * POSES_PER_COMPOUND))
    return synth.concat(parts)


def config1_slice():
    """BASELINE config 1: 1,024 poses, pocket 1,000 atoms, ligands <= 64 atoms."""
    from paper_2104_04547_b200 import synth
    pocket = synth.make_pocket(POCKET_ATOMS, seed=0)
    lib = synth.make_poses(103, POSES_PER_COMPOUND, seed=1, ligand_atoms=LIGAND_ATOMS).slice(0, 1024)
    return pocket, lib


# ---------------------------------------------------------------------------
# CPU oracle (the reference algorithm restated in numpy): config-1 slice
# ---------------------------------------------------------------------------
def _cpu_worker(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    s, e = args
    from oracle import fusion_oracle as orc
    from paper_2104_04547_b200 import synth
    from tests._cfg import COHERENT, GRAPH, VOXEL
    params = orc.init_params(VOXEL, GRAPH, COHERENT, 0)
    pocket, lib = config1_slice()
    t0 = time.perf_counter()
    out = [orc.score_pose(params, (VOXEL, GRAPH, COHERENT), *synth.complex_arrays(pocket, lib, p))["score"]
           for p in range(s, e)]
    return np.array(out), time.perf_counter() - t0


def cpu_oracle_pool(n_poses, workers):
    """Oracle scores of the first n_poses of the config-1 slice on `workers`
    processes x 1 BLAS thread; returns (scores, poses/s over the slowest)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    bounds = [(n_poses * i // workers, n_poses * (i + 1) // workers) for i in range(workers)]
    bounds = [b for b in bounds if b[1] > b[0]]
    with ctx.Pool(len(bounds)) as pool:
        res = pool.map(_cpu_worker, bounds)
    scores = np.concatenate([r[0] for r in res])
    return scores, n_poses / max(r[1] for r in res)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    """Reference arm: the reference algorithm (oracle port, float64 numpy) on
    all host cores; each step scores a bounded sample of the config-1 slice."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    workers = host_cores()
    per = 2
    t0 = time.perf_counter()
    for _ in range(args.warmup):
        cpu_oracle_pool(workers, workers)
    rates, times = [], []
    for _ in range(args.steps):
        s = time.perf_counter()
        rates.append(cpu_oracle_pool(workers * per, workers)[1])
        times.append(time.perf_counter() - s)
    value = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "poses/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "poses_per_step": workers * per},
            "cpu_baseline": {"value": value, "unit": "poses/s", "cores": workers, "kind": "port",
                             "sample": f"{workers} processes x {per} poses of the config-1 slice per step "
                                       "(oracle/fusion_oracle.py, float64, OPENBLAS_NUM_THREADS=1)"},
            "e2e": {"value": value, "unit": "poses/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t0}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm helpers
# ---------------------------------------------------------------------------
def _rel_stats(got, want):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    rel = np.abs(got - want) / np.abs(want)
    gc_, wc = got - got.mean(), want - want.mean()
    return {"max_rel": float(rel.max()), "median_rel": float(np.median(rel)),
            "max_abs": float(np.abs(got - want).max()),
            "centered_pearson": float(np.corrcoef(gc_, wc)[0, 1]),
            "max_centered_abs_over_spread": float(np.abs(gc_ - wc).max() / np.abs(wc).max())}


def _topk_idx(scores, k):
    s = np.asarray(scores, dtype=np.float64)
    return np.lexsort((np.arange(len(s)), -s))[:k]


def parity_config1(dm, E, precisions, workers):
    """Config 1 on the GPU (batch 32) vs the CPU oracle; the oracle pass is
    also the CPU baseline on all host cores."""
    pocket, lib = config1_slice()
    want, cpu_rate = cpu_oracle_pool(lib.n_poses, workers)
    pk = (pocket.xyz, pocket.elem, pocket.role, np.array([0, len(pocket.xyz)]))
    out = {"workload": "config1: 1,024 poses (pocket 1,000 atoms, ligands U{16..64}), batch 32, FusionModel(seed=0)",
           "oracle": "oracle/fusion_oracle.py (float64 numpy restatement, pinned to the reference goldens)"}
    k = 100
    want_top = _topk_idx(want, k)
    import torch
    for prec in precisions:
        got = []
        for s in range(0, lib.n_poses, 32):
            part = lib.slice(s, min(lib.n_poses, s + 32))
            b = E.batch_from_arrays(part.xyz, part.elem, part.role, part.atom_off, pocket=pk, pose_target=part.target)
            o = dm.score_poses(b, prec)
            got.append(o["scores"].cpu().numpy())
            assert not o["err"].cpu().numpy().any()
        torch.cuda.synchronize()
        got = np.concatenate(got)
        st = _rel_stats(got, want)
        top = _topk_idx(got, k)
        st["topk100_equal_oracle"] = bool(np.array_equal(top, want_top))
        st["topk100_overlap"] = len(set(top.tolist()) & set(want_top.tolist())) / k
        st["top10_equal_oracle"] = bool(np.array_equal(top[:10], want_top[:10]))
        out[prec] = st
    out["bars"] = {"fp32": "max_rel <= 1e-3", "mixed": "max_rel <= 1e-3",
                   "bf16": "max_rel <= 3e-3 and centered_pearson >= 0.9999 (stated; DESIGN.md section 4)"}
    out["pass"] = bool(out.get("fp32", {"max_rel": 0})["max_rel"] <= 1e-3 and
                       out.get("mixed", {"max_rel": 0})["max_rel"] <= 1e-3 and
                       out.get("bf16", {"max_rel": 0})["max_rel"] <= 3e-3)
    return out, cpu_rate, lib.n_poses


def precision_legs(dm, dlib, n_rank, bmax):
    """Throughput of the other precisions on the same screen (device-resident,
    eager calls of <= bmax poses): `mixed` (the 1e-3 path on tensor cores)
    over the whole shard, `fp32` (FFMA) over its first 16,384 poses.  Their
    accuracy vs the oracle is the `parity` block."""
    import torch
    out = {}
    for prec, n in (("mixed", n_rank), ("fp32", min(n_rank, 16384))):
        B = min(bmax, n)
        dm.score_poses(dlib.batch(0, min(B, 2048)), prec, 32768, retry=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        errs = []
        e0.record()
        for a in range(0, n, B):
            errs.append(dm.score_poses(dlib.batch(a, min(n, a + B)), prec, 32768, retry=False)["err"])
        e1.record()
        torch.cuda.synchronize()
        out[prec] = {"value": n / (e0.elapsed_time(e1) / 1e3), "unit": "poses/s", "poses": n,
                     "failed_poses": int(torch.cat(errs).ne(0).sum().item()),
                     "note": "same config-4 shard, device-resident, eager fs_score_poses calls (no top-k fold)"}
    return out


def plugin_legs(model_prec, dev):
    """End to end through the reference-facing API with host objects: the
    ModelScorer plugin (harness.py:224-234) with raw complexes, and
    predict_batch (models.py:470-498) with featurized items."""
    import torch
    from paper_2104_04547_b200 import complexes as cx
    from paper_2104_04547_b200 import harness, models, synth
    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    model = models.FusionModel(vcfg, gcfg, fcfg, seed=0, precision=model_prec)
    pocket = synth.make_pocket(POCKET_ATOMS, seed=0)
    lib = synth.make_poses(1700, POSES_PER_COMPOUND, seed=77, ligand_atoms=LIGAND_ATOMS)
    complexes = []
    for p in range(16384):
        pos, el, ro = synth.complex_arrays(pocket, lib, p)
        complexes.append(cx.SyntheticComplex(f"p{p}", pos, el, ro, 0.0))
    recs = [harness.PoseRecord(f"c{lib.compound[p]}", "t0", int(lib.pose_id[p]), complexes[p]) for p in range(16384)]
    scorer = harness.ModelScorer(model)
    out = {}

    def timed(fn, n_poses, reps=1):
        fn(n_poses)                              # warm: workspaces and pinned staging at full size
        torch.cuda.synchronize()
        best = None
        for _ in range(reps):
            t0 = time.perf_counter()
            fn(n_poses)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        return n_poses / best

    for bs, n in ((56, 4032), (16384, 16384)):
        def run(m, bs=bs):
            for s in range(0, m, bs):
                scorer(recs[s:min(m, s + bs)])
        rate = timed(run, n)
        atoms = sum(len(c.positions) for c in complexes[:bs])
        out[f"model_scorer_raw_b{bs}"] = {
            "value": rate, "unit": "poses/s", "poses": n,
            "h2d_bytes_per_call": int(atoms * (24 + 8 + 8) + (bs + 1) * 8), "d2h_bytes_per_call": 4 * bs + 4 * bs,
            "source": "harness.ModelScorer(list[PoseRecord]) with SyntheticComplex payloads (host numpy "
                      "vstack([pocket, ligand])), featurized on device in the call; wall clock incl. host work"}
    # the caller the reference actually uses: run_campaign drives the plugin
    # from a thread pool (harness.py:348-424), default batch 56; each scorer
    # thread runs on its own CUDA stream
    for par in (1, 4):
        sub = recs[:8064]
        harness.run_campaign(sub[:1008], scorer, n_jobs=4, parallelism=par, ranks_per_job=1, batch_size=56)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        preds, rep = harness.run_campaign(sub, scorer, n_jobs=16, parallelism=par, ranks_per_job=1, batch_size=56)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[f"run_campaign_raw_b56_threads{par}"] = {
            "value": len(preds) / dt, "unit": "poses/s", "poses": len(preds), "complete": rep.complete,
            "source": f"harness.run_campaign(16 jobs, parallelism={par}, batch 56) -> ModelScorer with raw "
                      "SyntheticComplex payloads; wall clock of the whole campaign"}
    items = models.featurize(complexes[:2048], vcfg, gcfg)
    pairs = [(it.grid, it.graph) for it in items]
    for bs in (56, 2048):
        def run(m, bs=bs):
            for s in range(0, m, bs):
                model.predict_batch(pairs[s:min(m, s + bs)])
        n = 2016 if bs == 56 else 2048
        rate = timed(run, n)
        g = pairs[0][1]
        per_pose = 8 * 4096 * 8 + np.asarray(g.node_features).nbytes + 16 * (len(g.covalent_edges) +
                                                                             len(g.noncovalent_edges))
        out[f"predict_batch_featurized_b{bs}"] = {
            "value": rate, "unit": "poses/s", "poses": n, "h2d_bytes_per_pose": int(per_pose),
            "source": "FusionModel.predict_batch([(VoxelGrid, ComplexGraph)]): host validation in the reference's "
                      "order, float64 grids + features + edges staged through pinned memory; wall clock"}
    return out


def config_legs(dm, E, N, dev, precision):
    """BASELINE configs 2, 3 and 5 (device-timed with CUDA events)."""
    import torch
    from oracle import radius_c
    from paper_2104_04547_b200 import synth
    out = {}
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # ---- config 2: featurizer only (the drop-in featurize outputs: float64
    # voxel grids + canonical edge lists with float64 distances) ----
    pocket = synth.make_pocket(POCKET_ATOMS, seed=5)
    lib2 = screen_library(0, 10_000, seed=500)
    pk = (pocket.xyz, pocket.elem, pocket.role, np.array([0, POCKET_ATOMS]))
    B2 = 12_500
    batches = [E.batch_from_arrays(lib2.xyz[lib2.atom_off[s]:lib2.atom_off[s + B2]], lib2.elem[lib2.atom_off[s]:
                                   lib2.atom_off[s + B2]], lib2.role[lib2.atom_off[s]:lib2.atom_off[s + B2]],
                                   lib2.atom_off[s:s + B2 + 1] - lib2.atom_off[s], pocket=pk,
                                   pose_target=lib2.target[s:s + B2]) for s in range(0, lib2.n_poses, B2)]

    def featurize(b):
        grids, err = E.voxelize(b, 16, 4, 16.0)
        g = E.radius_graph(b, 2.24, 5.22, with_dists=True)
        ce = E.edge_lists(g, "cov")
        ne = E.edge_lists(g, "ncov")
        return grids, g, ce, ne
    featurize(batches[0])
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    for b in batches:
        res = featurize(b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # bit-exactness on a 1,000-pose sample of the last batch vs the C oracle
    grids, g, (ce, cd, coff), (ne, nd, noff) = res
    S = 1000
    s0 = lib2.n_poses - B2
    part = lib2.slice(s0, s0 + S)
    lig = np.diff(part.atom_off)
    off = np.concatenate([[0], np.cumsum(lig + POCKET_ATOMS)]).astype(np.int64)
    pos = np.concatenate([np.vstack([pocket.xyz, part.xyz[part.atom_off[p]:part.atom_off[p + 1]]]) for p in range(S)])
    roles = np.concatenate([np.r_[np.zeros(POCKET_ATOMS, np.int64), np.ones(lig[p], np.int64)] for p in range(S)])
    wce, wcd, wcoff, wne, wnd, wnoff = radius_c.radius_pairs_batch(pos, roles, off)
    ok = True
    for (edges, dists, eoff), (we, wd, woff) in (((ce, cd, coff), (wce, wcd, wcoff)), ((ne, nd, noff), (wne, wnd, wnoff))):
        eo = eoff[: S + 1].cpu().numpy()
        ok &= np.array_equal(edges[: eo[-1]].cpu().numpy(), we) and np.array_equal(
            dists[: eo[-1]].cpu().numpy().view(np.uint64), wd.view(np.uint64)) and np.array_equal(eo, woff)
    out["config2_featurize"] = {
        "value": lib2.n_poses / (ms / 1e3), "unit": "poses/s", "poses": lib2.n_poses,
        "edges_bitwise_vs_oracle_sample": bool(ok), "sample": f"{S} poses vs oracle/radius_graph.c",
        "note": "featurizer API path (voxelize float64 NCDHW + count/fill radius graph + canonical edge lists "
                "with float64 distances, what featurize returns); the scoring path fuses a leaner graph into "
                "fs_score_poses; all 100,000 poses of the config timed (8 batches of 12,500)"}

    # ---- config 3: each branch alone on featurized input, batch 256 ----
    B3 = 256
    n_inputs = 4                                    # distinct 256-pose batches, round robin (> L2)
    lib3 = screen_library(0, 103, seed=900).slice(0, B3 * n_inputs)
    inputs = []
    for i in range(n_inputs):
        part = lib3.slice(i * B3, (i + 1) * B3)
        b = E.batch_from_arrays(part.xyz, part.elem, part.role, part.atom_off, pocket=pk, pose_target=part.target)
        grids, _ = E.voxelize(b, 16, 4, 16.0)
        g = E.radius_graph(b, 2.24, 5.22, with_dists=False)
        feats = E.node_features(b, g.node_off, 4, 16.0)
        ce, _, coff = E.edge_lists(g, "cov")
        ne, _, noff = E.edge_lists(g, "ncov")
        no = g.node_off
        # edge lists are pose-local: lift them to global node ids
        cp = torch.repeat_interleave(torch.arange(B3, device=dev), coff.diff())
        np_ = torch.repeat_interleave(torch.arange(B3, device=dev), noff.diff())
        inputs.append((grids, feats, no, ce + no[cp][:, None], ne + no[np_][:, None], int(no.diff().max().item())))
    for prec, n_batches in (("bf16", 391), ("fp32", 391)):
        for head, name in ((1, "voxel"), (2, "graph")):
            def once(i):
                grids, feats, no, ce, ne, mpn = inputs[i % n_inputs]
                if head == 1:
                    dm.score_features(B3, grids=grids, heads=1, precision=prec, max_pose_nodes=0)
                else:
                    dm.score_features(B3, feats=feats, node_off=no, cov_edges=ce, ncov_edges=ne, heads=2,
                                      precision=prec, max_pose_nodes=mpn)
            once(0)
            torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record()
            for i in range(n_batches):
                once(i)
            e1.record()
            torch.cuda.synchronize()
            out[f"config3_{name}_head_{prec}"] = {
                "value": n_batches * B3 / (e0.elapsed_time(e1) / 1e3), "unit": "poses/s", "poses": n_batches * B3,
                "batch": B3, "precision": prec}
    out["config3_note"] = ("branch-alone forwards (voxel_head_forward / graph_head_forward semantics) on featurized "
                           "device input, 4 distinct 256-pose batches round robin; 100,096 poses timed per "
                           "head and precision")

    # ---- config 5: 4 targets, variable ligand sizes ----
    tgts = synth.FOUR_TARGETS
    pockets = [synth.make_pocket(n, seed=40 + i, name=nm) for i, (nm, n) in enumerate(tgts)]
    B5, K5 = 32768, 38                             # 1,245,184 poses: one GPU's share of 10M over 8
    per_t = B5 * K5 // len(tgts)
    libs = [screen_library(0, (per_t + 9) // 10, seed=4000 + 100 * i, ligand_atoms=(8, 96), target=i).slice(0, per_t)
            for i in range(len(tgts))]
    for i, l in enumerate(libs):
        l.compound = l.compound + i * 10_000_000
    from paper_2104_04547_b200.screen import DeviceLibrary
    lib5 = synth.concat(libs)                      # target by target, as a campaign screens them
    dlib5 = DeviceLibrary(lib5, pockets, dev)
    dm.score_poses(dlib5.batch(0, B5), precision, 32768, retry=False)
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    top = (None, None)
    errs = []
    for i in range(K5):
        o = dm.score_poses(dlib5.batch(i * B5, (i + 1) * B5), precision, 32768, retry=False)
        top = E.topk_merge(top[0], top[1], o["scores"], dlib5.pidx[i * B5:(i + 1) * B5], TOPK)
        errs.append(o["err"])
    e1.record()
    torch.cuda.synchronize()
    out["config5_four_targets"] = {
        "value": B5 * K5 / (e0.elapsed_time(e1) / 1e3), "unit": "poses/s", "poses": B5 * K5,
        "failed_poses": int(torch.stack(errs).ne(0).sum().item()), "precision": precision,
        "targets": {nm: n for nm, n in tgts}, "ligand_atoms": [8, 96],
        "note": "4 synthetic pockets (protease1/2 = 1000/900 atoms, spike1/2 = 450/350, SURVEY 8d proposal); "
                "1,245,184 poses timed on this GPU (the config's 10M over 8 GPUs is 1.25M per GPU)"}
    return out


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--precision", default=os.environ.get("FS_BENCH_PRECISION", "bf16"))
    ap.add_argument("--scaling", default="strong", choices=("strong", "weak"))
    ap.add_argument("--batch", type=int, default=int(os.environ.get("FS_BENCH_BATCH", "16384")),
                    help="poses per step per rank for --scaling weak")
    ap.add_argument("--screen-compounds", type=int, default=SCREEN_COMPOUNDS)
    ap.add_argument("--no-extras", action="store_true", help="skip parity/plugin/configs legs")
    ap.add_argument("--no-factored", action="store_true", help="skip the pocket-factored effective-throughput leg")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    # NCCL's version banner goes to stdout at NCCL_DEBUG=VERSION/WARN: route
    # every NCCL message to stderr so stdout stays the one JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import torch
    import torch.distributed as dist
    from paper_2104_04547_b200 import _native as N
    from paper_2104_04547_b200 import engine as E
    from paper_2104_04547_b200 import harness, models, poselib, synth
    from paper_2104_04547_b200.screen import DeviceLibrary, compound_topk, merge_topk_across_ranks

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    vcfg, gcfg, fcfg = models.VoxelHeadConfig(), models.GraphHeadConfig(), models.table_coherent_fusion_config()
    model = models.FusionModel(vcfg, gcfg, fcfg, seed=0)
    dm = E.DeviceModel(vcfg, gcfg, fcfg, model.all_params(), device=dev)
    precision = args.precision
    if not dm.supports(precision):
        precision = "fp32"
    K, W = args.steps, args.warmup

    # ---- this rank's shard ----
    if args.scaling == "strong":
        n_comp_total = args.screen_compounds
        c0, c1 = harness.shard_bounds(n_comp_total, world)[rank]
        B = max(1, math.ceil((c1 - c0) * POSES_PER_COMPOUND / K))
    else:
        B = args.batch
        per = (K * B + POSES_PER_COMPOUND - 1) // POSES_PER_COMPOUND
        n_comp_total = per * world
        c0, c1 = rank * per, (rank + 1) * per
    lib = screen_library(c0, c1, seed=1)
    if args.scaling == "weak":
        lib = lib.slice(0, K * B)
    n_rank = lib.n_poses
    pocket = synth.make_pocket(POCKET_ATOMS, seed=0)
    dlib = DeviceLibrary(lib, [pocket], dev, index_base=c0 * POSES_PER_COMPOUND)
    L = N.lib()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    bounds = [(min(n_rank, i * B), min(n_rank, (i + 1) * B)) for i in range(K)]
    BMAX = int(os.environ.get("FS_BENCH_BMAX", "32768"))   # poses per fs_score_poses call (workspace ~0.6 MB/pose)
    n_comp = c1 - c0

    # one set of stage events per fs_score_poses call (a step is one or more calls)
    calls = [(a, min(e, a + BMAX)) for s, e in bounds for a in range(s, e, BMAX)]
    stage_events = {c: [torch.cuda.Event(enable_timing=True) for _ in N.STAGES] for c in calls}
    for evs in stage_events.values():   # torch creates CUDA events lazily: force creation
        for e in evs:
            e.record()
    ev_ptrs = {c: (E.C.c_void_p * len(evs))(*[E.C.c_void_p(e.cuda_event) for e in evs])
               for c, evs in stage_events.items()}

    def score_call(scoref, a, b):
        L.fs_set_stage_events(ev_ptrs[(a, b)], len(N.STAGES))
        out = scoref(a, b)
        L.fs_set_stage_events(None, 0)
        return out

    def step(s, e, top, acc):
        # one screening step: featurize + score the batch (in calls of at
        # most BMAX poses), fold it into the running pose top-k and the
        # per-compound best pose (all on device)
        for a in range(s, e, BMAX):
            b = min(e, a + BMAX)
            out = score_call(lambda x, y: dm.score_poses(dlib.batch(x, y), precision, 32768, retry=False), a, b)
            top = E.topk_merge(top[0], top[1], out["scores"], dlib.pidx[a:b], TOPK)
            acc.update(dlib.compound[a:b], dlib.pose_id[a:b], out["scores"])
        return out, top

    def finish(top, acc):
        gs, gi = merge_topk_across_ranks(top[0], top[1], TOPK, device=dev)
        ct = compound_topk(acc, TOPK)
        cs, ci = merge_topk_across_ranks(ct["topk_compound_scores"], ct["topk_compound_idx"], TOPK, device=dev)
        return gi, ci

    # ---- warm-up (also validates: no pose may fail) ----
    top = (None, None)
    acc = E.BestPoseAccumulator(n_comp, c0, device=dev)
    for i in range(W):
        s, e = bounds[i % K]
        out, top = step(s, e, top, acc)
    torch.cuda.synchronize()
    assert int(out["err"].abs().sum().item()) == 0, "pose errors in warm-up batch"

    def run_steps(stepf):
        top = (None, None)
        acc = E.BestPoseAccumulator(n_comp, c0, device=dev)
        errs = []
        for i in range(K):
            flush.zero_()                                  # L2 flush between steps
            s, e = bounds[i]
            out, top = stepf(s, e, top, acc)
            errs.append(out["err"])
        return top, acc, errs

    def capture(stepf):
        """The K steps as one CUDA graph (host stalls cannot idle the GPU, no
        per-launch overhead); None if capture is not possible here."""
        if os.environ.get("FS_BENCH_EAGER"):
            return None
        try:
            graph = torch.cuda.CUDAGraph()
            n0 = L.fs_launch_count()
            with torch.cuda.graph(graph):
                res = run_steps(stepf)
            n_launch = L.fs_launch_count() - n0
            graph.replay()                                 # warm replay
            torch.cuda.synchronize()
            return graph, res, n_launch
        except Exception as exc:                           # noqa: BLE001 -- fall back to eager
            print(f"bench: CUDA graph capture unavailable ({exc}); timing eagerly", file=sys.stderr)
            torch.cuda.synchronize()
            return None

    def stage_sum(only=None):
        tot = np.zeros(len(N.STAGES) - 1)
        for c in (only or calls):
            evs = stage_events[c]
            for j in range(len(N.STAGES) - 1):
                tot[j] += evs[j].elapsed_time(evs[j + 1])
        return tot

    # ---- timed region: device-resident inputs ----
    cap = capture(step)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.fs_launch_count()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gc.disable()
    with Clocks(local) as clk:
        clk.ready()
        t_start.record()
        if cap is not None:
            graph, (top, acc, errs), launches = cap
            graph.replay()
        else:
            top, acc, errs = run_steps(step)
        gi, gci = finish(top, acc)
        t_end.record()
        torch.cuda.synchronize()
    graphed = cap is not None
    launches = launches if graphed else L.fs_launch_count() - launches0
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end)
    stage_ms = stage_sum()
    bad = int(torch.cat(errs).ne(0).sum().item())
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_poses = torch.tensor([n_rank], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(total_poses)
    total_poses = int(total_poses.item())
    value = total_poses / (ms_max / 1e3)
    del cap
    torch.cuda.synchronize()

    # ---- serial per-kernel timing (exact stage events; same results) ----
    L.fs_set_overlap(0)
    top_s = (None, None)
    acc_s = E.BestPoseAccumulator(n_comp, c0, device=dev)
    serial_calls = [c for c in calls if c[1] > c[0]][:3]
    for a, b in serial_calls:
        flush.zero_()
        _, top_s = step(a, b, top_s, acc_s)
        torch.cuda.synchronize()
    serial = stage_sum(serial_calls)
    L.fs_set_overlap(-1)
    serial_poses = sum(b - a for a, b in serial_calls)

    # ---- end to end: packed library file (memory-mapped) -> pinned double
    # buffer -> H2D on a copy stream overlapping the previous batch's scoring;
    # every step's scores are read back to pinned host memory ----
    lib_path = os.path.join(tempfile.gettempdir(), f"fs_bench_lib_r{rank}_{os.getpid()}.fspl")
    poselib.save_library(lib_path, [pocket], lib)
    pk_m, lib_m = poselib.load_library(lib_path)
    BE = min(B, BMAX)
    loader = poselib.StreamingLoader(lib_m, pk_m, BE, dev, index_base=c0 * POSES_PER_COMPOUND)
    h_scores = torch.empty(BE, dtype=torch.float32).pin_memory()
    e2e_batches = math.ceil(bounds[-1][1] / BE)

    def e2e_pass(n_batches):
        top, acc, d2h = (None, None), E.BestPoseAccumulator(n_comp, c0, device=dev), 0
        for i, (s, e, b, comp, pid) in enumerate(loader.batches(BE)):
            if i == n_batches:
                break
            o = dm.score_poses(b, precision, 32768, retry=False)
            top = E.topk_merge(top[0], top[1], o["scores"], dlib.pidx[s:e], TOPK)
            acc.update(comp, pid, o["scores"])
            h_scores[: e - s].copy_(o["scores"], non_blocking=True)
            d2h += (e - s) * 4
        return top, acc, d2h

    e2e_pass(min(W, e2e_batches))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    loader.h2d_bytes = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    top2, acc2, d2h = e2e_pass(e2e_batches)
    gi2, gci2 = finish(top2, acc2)
    e1.record()
    torch.cuda.synchronize()
    h2d = loader.h2d_bytes
    os.unlink(lib_path)
    te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = total_poses / (float(te.item()) / 1e3)
    same_topk = bool(torch.equal(gi, gi2)) and bool(torch.equal(gci, gci2))

    # ---- pocket-invariant factoring: effective throughput of
    # the same screen, reported beside (not instead of) the full path ----
    fact = None
    if precision in ("bf16", "mixed") and not args.no_factored:
        t0 = time.perf_counter()
        cache = dm.prepare_pockets(dlib.pocket_xyz, dlib.pocket_elem, dlib.pocket_role, dlib.pocket_off,
                                   precision=precision)
        torch.cuda.synchronize()
        prep_ms = (time.perf_counter() - t0) * 1e3

        def fstep(s, e, top, acc):
            for a in range(s, e, BMAX):
                b = min(e, a + BMAX)
                out = score_call(lambda x, y: dm.score_poses_cached(dlib.batch(x, y), cache, 32768, rescore=False),
                                 a, b)
                top = E.topk_merge(top[0], top[1], out["scores"], dlib.pidx[a:b], TOPK)
                acc.update(dlib.compound[a:b], dlib.pose_id[a:b], out["scores"])
            return out, top

        top = (None, None)
        acc = E.BestPoseAccumulator(n_comp, c0, device=dev)
        for i in range(W):
            s, e = bounds[i % K]
            out_f, top = fstep(s, e, top, acc)
        nb0 = min(B, BMAX)
        ref_full = dm.score_poses(dlib.batch(0, nb0), precision, 32768, retry=False)["scores"]
        ref_fact = fstep(0, nb0, (None, None), acc)[0]["scores"]
        torch.cuda.synchronize()
        fact_err = int(out_f["err"].ne(0).sum().item())
        max_diff = float((ref_full - ref_fact).abs().max().item())
        fcap = capture(fstep)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        if fcap is not None:
            fgraph, (top, acc, _), _ = fcap
            fgraph.replay()
        else:
            top, acc, _ = run_steps(fstep)
        gi_f, gci_f = finish(top, acc)
        f1.record()
        torch.cuda.synchronize()
        fstage = stage_sum()
        tf = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tf, op=dist.ReduceOp.MAX)
        fact = {"value": total_poses / (float(tf.item()) / 1e3), "unit": "poses/s",
                "ms_per_step": float(tf.item()) / K, "prepare_ms_per_pocket": prep_ms,
                "stage_ms_per_step": {n: round(v / K, 4) for n, v in zip(N.STAGES[:-1], fstage)},
                "max_abs_score_diff_vs_full_path": max_diff, "failed_poses": fact_err,
                "topk_equal_full_path": bool(torch.equal(gi, gi_f)),
                "topk_overlap_full_path": len(set(gi.tolist()) & set(gi_f.tolist())) / max(1, gi.numel()),
                "compound_topk_equal_full_path": bool(torch.equal(gci, gci_f)),
                "note": "effective throughput: pocket-invariant work (pocket conv1 channels, pocket covalent "
                        "phase, untouched pocket nodes) reused from a per-target cache; algorithmic work per "
                        "pose and the roofline are those of the full path (SURVEY 8d/8f-4)"}
        del fcap, cache

    # mean nodes / edges of this workload (for the algorithmic FLOP formula)
    sample = dlib.batch(0, min(n_rank, 2048))
    gr = E.scoring_graph_entries(sample, 2.24, 5.22, 32768, with_dists=False)
    ec_mean = float(gr["n_cov"].double().mean().item()) / 2
    en_mean = float(gr["n_ncov"].double().mean().item()) / 2
    del gr
    n_mean = POCKET_ATOMS + float(np.mean(np.diff(lib.atom_off)))

    gc.enable()
    extras = {}
    if rank == 0 and world == 1 and not args.no_extras:
        torch.cuda.empty_cache()
        extras["parity"], cpu_rate, cpu_n = parity_config1(dm, E, ("fp32", "mixed", "bf16"), host_cores())
        extras["cpu_baseline"] = {"value": cpu_rate, "unit": "poses/s", "cores": host_cores(), "kind": "port",
                                  "sample": f"config-1 slice ({cpu_n} poses: pocket 1,000 atoms, ligands <= 64) "
                                            "through oracle/fusion_oracle.py (float64 numpy), one process per "
                                            "host core x 1 BLAS thread; rate over the slowest process"}
        # auxiliary legs never take the headline line down with them
        for key, fn in (("precisions", lambda: precision_legs(dm, dlib, n_rank, BMAX)),
                        ("plugin", lambda: plugin_legs(precision, dev)),
                        ("configs", lambda: config_legs(dm, E, N, dev, precision))):
            try:
                extras[key] = fn()
            except Exception as exc:                   # noqa: BLE001
                torch.cuda.synchronize()
                extras[key] = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        hbm, bf16_burst, bf16_sus, peak_kind = peaks()
        names = N.STAGES[:-1]
        per_pose_ms = serial / max(1, serial_poses)             # exact per-kernel (serial pass)
        gflop = graph_flop(n_mean, ec_mean, en_mean)
        kern = {}
        for j, nm in enumerate(names):
            t_s = per_pose_ms[j] / 1e3
            if t_s <= 0:
                continue
            if nm in CONV_FLOP:
                kern[nm] = {"bound": "tensor", "achieved": CONV_FLOP[nm] / t_s / 1e12, "peak": bf16_burst,
                            "unit": "TFLOP/s", "issued_flop_frac": round(CONV_ISSUED[nm], 4),
                            "issued_tflops": CONV_ISSUED[nm] * CONV_FLOP[nm] / t_s / 1e12}
            elif nm == "gnn":
                kern[nm] = {"bound": "tensor", "achieved": gflop / t_s / 1e12, "peak": bf16_sus, "unit": "TFLOP/s"}
            elif nm == "dense":
                kern[nm] = {"bound": "hbm", "achieved": (4 * 4096 + 4 * 128) / t_s / 1e9, "peak": hbm,
                            "unit": "GB/s"}
            elif nm == "featurize":
                # voxel splat + fused radius graph: atoms in, bf16 grid + CSR out
                byt = 14 * n_mean + 2 * 8 * 4096 + 2 * 2 * (ec_mean + en_mean) + 8 * 2 * n_mean + 4 * 8 * n_mean
                kern[nm] = {"bound": "hbm", "achieved": byt / t_s / 1e9, "peak": hbm, "unit": "GB/s"}
            if nm in kern:
                kern[nm]["frac"] = kern[nm]["achieved"] / kern[nm]["peak"]
                kern[nm]["ms_per_16384_poses"] = round(per_pose_ms[j] * 16384, 4)
        dom = int(np.argmax(serial))
        dom_name = names[dom]
        ms_per_pose_timed = stage_ms[dom] / n_rank          # the timed run's own stage events
        gk = {"bf16": "gnn_mma_kernel<2> (GRU message passing on mma.sync: fp16 hi/lo activations x fp16 weights)",
              "mixed": "gnn_mma_kernel<3> (GRU message passing on mma.sync: bf16 hi/lo x hi/lo, 3 passes)",
              "fp32": "gnn_kernel (GRU message passing, FFMA fp32)"}[precision]
        if dom_name == "gnn":
            roof = {"kernel": gk, "bound": "tensor", "achieved": gflop / (ms_per_pose_timed / 1e3) / 1e12,
                    "peak": bf16_sus, "unit": "TFLOP/s", "traffic": None}
        elif dom_name in CONV_FLOP:
            roof = {"kernel": f"{dom_name} conv_umma_kernel", "bound": "tensor",
                    "achieved": CONV_FLOP[dom_name] / (ms_per_pose_timed / 1e3) / 1e12, "peak": bf16_sus,
                    "unit": "TFLOP/s", "traffic": None}
        else:
            roof = dict(kern.get(dom_name, {"bound": "tensor", "achieved": 0.0, "peak": bf16_sus, "unit": "TFLOP/s"}))
            roof["kernel"] = dom_name
            roof["traffic"] = None
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")))
            key = {"gnn": "gnn", "conv1": "conv1", "conv2": "conv2", "featurize": "graph_csr"}.get(dom_name)
            ent = tr.get(f"{key}_{precision}") or tr.get(key)
            if ent:
                roof["traffic"] = ent["bytes_per_pose"] * min(B, BMAX)
                roof["traffic_unit"] = f"bytes per launch ({min(B, BMAX)} poses)"
                roof["traffic_source"] = ("profiles/r02/ncu_traffic.json: ncu --set full dram__bytes_read.sum + "
                                          "dram__bytes_write.sum, per pose, scaled to this launch")
                if "onchip" in ent:
                    roof["onchip"] = ent["onchip"]
        except (OSError, ValueError):
            pass
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["peak_kind"] = f"{peak_kind} bf16 sustained (a kernel inside a long step)"
        roof["stage_ms_per_step"] = {n: round(v / K, 4) for n, v in zip(names, stage_ms)}
        roof["stage_note"] = ("per-step stage events of the overlapped timed run (the voxel branch runs on a side "
                              "stream beside the radius graph, so featurize/conv/dense are cross-stream deltas; "
                              "gnn is exact); per_kernel comes from a serial pass of the same steps")
        roof["dominant_share"] = float(serial[dom] / serial.sum())
        roof["per_kernel"] = kern
        roof["work_per_pose"] = {"nodes": n_mean, "cov_edges": ec_mean, "ncov_edges": en_mean,
                                 "graph_flop": gflop, "voxel_flop": VOXEL_FLOP}
        line = {"metric": METRIC, "value": value, "unit": "poses/s", "n_gpus": world, "steps": K, "warmup": W,
                "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": precision, "data": "synthetic",
                "config": {"workload": WORKLOAD if args.scaling == "strong" else WORKLOAD.replace(
                               "1,000,000 poses", f"{K}x{B} poses per rank"),
                           "screen_poses": total_poses, "poses_per_step_per_gpu": B, "precision": precision,
                           "topk": TOPK, "step": "featurize + score the rank's next batch, fold into pose top-k and "
                           "per-compound best pose on device; compound top-k + cross-rank NCCL merge after step K",
                           "pocket_atoms": POCKET_ATOMS, "ligand_atoms": list(LIGAND_ATOMS),
                           "l2": "256 MiB buffer zeroed between steps (inside the timed region)",
                           "weights": "random-init FusionModel(seed=0)", "failed_poses": bad},
                "roofline": roof,
                "e2e": {"value": e2e_value, "unit": "poses/s", "h2d_bytes_per_step": h2d // K,
                        "d2h_bytes_per_step": d2h // K, "topk_equal_device_resident": same_topk,
                        "source": "packed library file (mmap) -> pinned double buffer -> H2D on a copy stream; "
                                  "scores D2H every step"},
                "gpu_launches": int(launches), "clocks": clk.summary(),
                "launch_mode": "cuda_graph (K steps captured once, replayed in the timed region)" if graphed
                else "eager"}
        if fact is not None:
            line["pocket_factored"] = fact
        line.update(extras)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
