"""NCCL world-size-2 (and 4) correctness of the multi-GPU screen (SURVEY.md
8e(i)): the merged per-rank top-k over poses and compounds equals a
single-device sort of all scores, bitwise; a rank with an empty shard still
joins the collective.  Needs >= 2 GPUs (gpurun --gpus 2); skipped otherwise."""

import json
import os
import socket
import subprocess
import sys
import tempfile

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, compounds):
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(HERE, "_nccl_worker.py")]
    with tempfile.TemporaryDirectory() as out:
        # one result file per rank (the ranks' stdout lines can interleave)
        env = dict(os.environ, FS_TEST_COMPOUNDS=str(compounds), FS_TEST_OUT=out, NCCL_DEBUG_FILE="/dev/stderr")
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
        assert r.returncode == 0, r.stderr[-3000:]
        res = []
        for f in sorted(os.listdir(out)):
            with open(os.path.join(out, f)) as fh:
                res.append(json.load(fh))
    assert len(res) == world
    return sorted(res, key=lambda x: x["rank"])


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_topk_merge_equals_single_device_sort(world):
    res = _run(world, 301)
    assert res[0]["pose_topk_equal"] and res[0]["compound_topk_equal"], res[0]


def test_nccl_empty_shard_does_not_hang():
    res = _run(2, 1)                  # one compound: rank 1's shard is empty
    assert res[1]["shard"][0] == res[1]["shard"][1]
    assert res[0]["pose_topk_equal"] and res[0]["compound_topk_equal"], res[0]
