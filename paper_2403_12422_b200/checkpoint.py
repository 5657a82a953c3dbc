"""On-disk formats shared with the reference.

* ``int8flow-checkpoint-v1`` (``qlayers.py:598-637``): FP32 parameters as one
  little-endian float32 blob in sorted key order + a JSON manifest of shapes.
  ``save_params`` writes byte-identical files to the reference's; either side
  loads the other's checkpoints.
* Training state as the reference trainer stores it (``trainer.py:462-477,
  526-536``): keys ``param.<k>``, ``m.<k>``, ``v.<k>`` + manifest ``step``,
  ``opt_t``, ``scheme`` — resumable here or by ``int8flow.run_training``.
* JQT1 ``BlockQuantTensor`` blobs live on ``BlockQuantTensor.to_bytes /
  from_bytes`` (``qtensor.py:152-181``).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import torch

FORMAT = "int8flow-checkpoint-v1"


def _host_f32(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        a = a.detach().to("cpu", torch.float32).numpy()
    return np.ascontiguousarray(a, dtype="<f4")


def save_params(path, params: dict, manifest: dict | None = None) -> None:
    """Write ``<path>.bin`` + ``<path>.json`` exactly as ``int8flow.qlayers.save_params``."""
    path = Path(path)
    keys = sorted(params)
    shapes = {k: list(params[k].shape) for k in keys}
    blob = b"".join(_host_f32(params[k]).tobytes() for k in keys)
    path.with_suffix(".bin").write_bytes(blob)
    doc = {"format": FORMAT, "params": shapes, "manifest": manifest or {}}
    path.with_suffix(".json").write_text(json.dumps(doc, indent=2, sort_keys=True))


def load_params(path) -> tuple[dict, dict]:
    """(params as float32 numpy arrays, manifest); the reference's errors for bad files."""
    path = Path(path)
    doc = json.loads(path.with_suffix(".json").read_text())
    if doc.get("format") != FORMAT:
        raise ValueError(f"unrecognized checkpoint format: {doc.get('format')!r}")
    blob = path.with_suffix(".bin").read_bytes()
    params, offset = {}, 0
    for key in sorted(doc["params"]):
        shape = tuple(doc["params"][key])
        count = int(np.prod(shape)) if shape else 1
        params[key] = np.frombuffer(blob, dtype="<f4", count=count, offset=offset).reshape(shape).astype(np.float32)
        offset += 4 * count
    if offset != len(blob):
        raise ValueError("checkpoint blob size does not match manifest shapes")
    return params, doc["manifest"]


def save_training_state(path, model, opt, step: int) -> None:
    """Parameters + AdamW moments in the reference trainer's layout."""
    state = {}
    for k, p in model.params.items():
        state[f"param.{k}"] = p
        state[f"m.{k}"] = opt.m[k]
        state[f"v.{k}"] = opt.v[k]
    save_params(path, state, {"step": int(step), "opt_t": int(opt.t), "scheme": "per-block"})


def load_training_state(path, model, opt) -> int:
    """Restore parameters + moments (trainer.py:462-477); returns the checkpoint step."""
    state, meta = load_params(path)
    for k, p in model.params.items():
        p.copy_(torch.from_numpy(state[f"param.{k}"]))
        opt.m[k].copy_(torch.from_numpy(state[f"m.{k}"]))
        opt.v[k].copy_(torch.from_numpy(state[f"v.{k}"]))
    opt.t = int(meta["opt_t"])
    model.mark_updated()
    return int(meta["step"])


__all__ = ["FORMAT", "load_params", "load_training_state", "save_params", "save_training_state"]
