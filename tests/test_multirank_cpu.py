"""World-size-2 gloo test of the multi-GPU host logic on CPU: compound-aligned
sharding, global pose indices, NaN padding, the all-gather of per-rank top-k
and the (score desc, index asc) merge -- everything but the device kernels."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def cpu_merge(s, i, k):
    s = s.double().numpy()
    i = i.numpy()
    key = np.where(np.isnan(s), np.inf, -s)
    order = np.lexsort((i, key))[:k]
    return torch.from_numpy(s[order].astype(np.float32)), torch.from_numpy(i[order])


def fake_scores(idx):
    # deterministic pseudo-scores with many exact ties
    return ((idx * 2654435761) % 97).astype(np.float32) / 97.0


def _worker(rank, world, port, k, out_q, n_comp=53):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2104_04547_b200 import harness, synth
    from paper_2104_04547_b200.screen import merge_topk_across_ranks
    lib = synth.make_poses(n_comp, poses_per_compound=10, seed=4)
    bounds = harness.compound_aligned_bounds(lib.compound, world)
    s, e = bounds[rank]
    idx = np.arange(s, e, dtype=np.int64)
    sc = fake_scores(idx)
    if e > s:
        ls, li = cpu_merge(torch.from_numpy(sc), torch.from_numpy(idx), k)
    else:                      # empty shard: still joins the collective
        ls = li = None
    gs, gi = merge_topk_across_ranks(ls, li, k, merge=cpu_merge, device=torch.device("cpu"))
    out_q.put((rank, gs.numpy(), gi.numpy(), (s, e)))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_two_rank_topk_merge_equals_single_sort():
    world, k = 2, 25
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    # shards tile the library and never split a compound
    assert res[0][3][0] == 0 and res[0][3][1] == res[1][3][0] and res[1][3][1] == 530
    # every rank holds the same merged top-k == single-device sort of all scores
    all_idx = np.arange(530, dtype=np.int64)
    ws, wi = cpu_merge(torch.from_numpy(fake_scores(all_idx)), torch.from_numpy(all_idx), k)
    for _, gs, gi, _ in res:
        assert np.array_equal(gi, wi.numpy())
        assert np.array_equal(gs, ws.numpy())


def test_empty_shard_joins_the_collective():
    """More ranks than compounds: a rank with an empty shard pads with NaN and
    still joins the all-gather (no hang); the merged top-k equals
    the single sort of all scores followed by the padding."""
    world, k = 2, 25
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, q, 1)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    assert res[1][3][0] == res[1][3][1]          # rank 1 owns no poses
    all_idx = np.arange(10, dtype=np.int64)
    ws, wi = cpu_merge(torch.from_numpy(fake_scores(all_idx)), torch.from_numpy(all_idx), k)
    for _, gs, gi, _ in res:
        assert np.array_equal(gi[:10], wi.numpy()) and np.array_equal(gs[:10], ws.numpy())
        assert np.isnan(gs[10:]).all() and (gi[10:] == np.iinfo(np.int64).max).all()
