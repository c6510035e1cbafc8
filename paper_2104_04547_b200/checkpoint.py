"""Reader/writer for the reference checkpoint container (checkpoint.py:21-71).

npz with ``param/<name>`` float64 arrays and a JSON ``__header__`` (uint8)
holding format_version, param_names and meta.  Optimizer state is read and
ignored (training is out of scope), so reference checkpoints load unchanged.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

FORMAT_VERSION = 1


def save_checkpoint(path, params: dict, meta: dict | None = None) -> None:
    payload = {f"param/{k}": np.asarray(v, dtype=np.float64) for k, v in params.items()}
    header = {"format_version": FORMAT_VERSION, "param_names": sorted(params), "meta": meta or {}}
    payload["__header__"] = np.frombuffer(json.dumps(header, sort_keys=True).encode(), dtype=np.uint8)
    with open(path, "wb") as f:
        np.savez(f, **payload)


def load_checkpoint(path):
    """Returns (params, meta) -- the reference returns (params, optimizer, meta)."""
    with np.load(Path(path)) as z:
        header = json.loads(bytes(z["__header__"]).decode())
        if header["format_version"] != FORMAT_VERSION:
            raise ValueError(f"unsupported checkpoint format {header['format_version']}")
        params = {n: np.array(z[f"param/{n}"]) for n in header["param_names"]}
    return params, header["meta"]
