"""Reader/writer for the reference checkpoint container (checkpoint.py:21-71).

npz with ``param/<name>`` float64 arrays, optional ``opt/<name>`` optimizer
state arrays, and a JSON ``__header__`` (uint8) holding format_version,
param_names, meta and (if saved) the optimizer's config and step count.
Same signatures as the reference: ``save_checkpoint(path, params, optimizer,
meta)`` and ``load_checkpoint(path) -> (params, optimizer, meta)``.

Training is outside the scoring path, so the optimizer comes back as an
:class:`OptimizerState` -- the reference Optimizer's config, step count and
state arrays, carried unchanged so a checkpoint round-trips bitwise -- rather
than a live optimizer.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

FORMAT_VERSION = 1

__all__ = ["save_checkpoint", "load_checkpoint", "FORMAT_VERSION", "OptimizerState"]


@dataclass
class OptimizerState:
    """Optimizer section of a checkpoint (checkpoint.py:32-41, :56-70)."""

    kind: str
    learning_rate: float
    coefficients: dict = field(default_factory=dict)
    step_count: int = 0
    arrays: dict = field(default_factory=dict)     # "<param>::<slot>" -> float64 array

    def state_arrays(self) -> dict:
        return self.arrays


def _opt_header(opt) -> tuple[dict, dict]:
    """(header dict, state arrays) of an OptimizerState or a reference-style
    optimizer (``.cfg.kind`` / ``.step_count`` / ``.state_arrays()``)."""
    if isinstance(opt, OptimizerState):
        head = {"kind": opt.kind, "learning_rate": opt.learning_rate, "coefficients": opt.coefficients,
                "step_count": opt.step_count}
    else:
        head = {"kind": opt.cfg.kind, "learning_rate": opt.cfg.learning_rate,
                "coefficients": opt.cfg.coefficients, "step_count": opt.step_count}
    return head, dict(opt.state_arrays())


def save_checkpoint(path, params: dict, optimizer=None, meta: dict | None = None) -> None:
    payload = {f"param/{k}": np.asarray(v, dtype=np.float64) for k, v in params.items()}
    header = {"format_version": FORMAT_VERSION, "param_names": sorted(params), "meta": meta or {}}
    if optimizer is not None:
        header["optimizer"], arrays = _opt_header(optimizer)
        for name, arr in arrays.items():
            payload[f"opt/{name}"] = arr
    payload["__header__"] = np.frombuffer(json.dumps(header, sort_keys=True).encode(), dtype=np.uint8)
    with open(path, "wb") as f:
        np.savez(f, **payload)


def load_checkpoint(path):
    """Returns (params, optimizer-or-None, meta), as the reference does."""
    with np.load(Path(path)) as z:
        header = json.loads(bytes(z["__header__"]).decode())
        if header["format_version"] != FORMAT_VERSION:
            raise ValueError(f"unsupported checkpoint format {header['format_version']}")
        params = {n: np.array(z[f"param/{n}"]) for n in header["param_names"]}
        optimizer = None
        if "optimizer" in header:
            o = header["optimizer"]
            arrays = {k[len("opt/"):]: np.array(z[k]) for k in z.files if k.startswith("opt/")}
            optimizer = OptimizerState(o["kind"], o["learning_rate"], dict(o["coefficients"]),
                                       int(o["step_count"]), arrays)
    return params, optimizer, header["meta"]
