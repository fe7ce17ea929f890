"""Policy parameters: names, shapes, init, flat device layout, checkpoint JSON.

Mirrors reference ``policy.py:70-98`` (names / shapes / Glorot draw order, so
``init_policy_params(config, seed)`` is bit-identical to the reference's) and
``nn.py:235-309`` (checkpoint format v1).  Parameters are float64 like the
reference; on the GPU they live in ONE flat float64 vector whose layout is the
sorted-name order of the checkpoint (``FlatLayout``).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

N_STATIC_FEATURES = 5
N_DEVICE_FEATURES = 5
N_DYNAMIC_COLS = 2
CHECKPOINT_VERSION = 1


class Param:
    """Minimal stand-in for the reference's ``nn.Tensor`` leaf: ``.data``
    (float64 ndarray), ``.grad``, ``.shape``; callers that mutate
    ``params[name].data`` keep working."""

    __slots__ = ("data", "grad", "requires_grad")

    def __init__(self, data, requires_grad: bool = True):
        self.data = np.atleast_2d(np.asarray(data, dtype=np.float64))
        self.grad = None
        self.requires_grad = requires_grad

    @property
    def shape(self) -> tuple[int, int]:
        return self.data.shape

    def __repr__(self) -> str:
        return f"Param(shape={self.shape})"


Params = dict  # name -> Param


def as_array(p) -> np.ndarray:
    return p.data if hasattr(p, "data") and not isinstance(p, np.ndarray) else np.asarray(p)


def glorot_uniform(rng: np.random.Generator, rows: int, cols: int) -> Param:
    a = math.sqrt(6.0 / (rows + cols))
    return Param(rng.uniform(-a, a, size=(rows, cols)))


def zeros_param(rows: int, cols: int) -> Param:
    return Param(np.zeros((rows, cols)))


def encoder_names(config) -> list[str]:
    return ["enc"] if config.shared_encoder else ["plc", "sel"]


def init_policy_params(config, seed: int = 0) -> Params:
    """Same draws in the same order as reference ``policy.py:74-98``."""
    rng = np.random.default_rng(seed)
    h = config.hidden
    p: Params = {}
    for enc in encoder_names(config):  # sorted order, as the reference
        d_prev = N_STATIC_FEATURES + N_DYNAMIC_COLS
        for k in range(config.k_rounds):
            p[f"{enc}.gnn{k}.psi.w"] = glorot_uniform(rng, 2 * d_prev + 1, h)
            p[f"{enc}.gnn{k}.psi.b"] = zeros_param(1, h)
            p[f"{enc}.gnn{k}.phi.w"] = glorot_uniform(rng, d_prev + h, h)
            p[f"{enc}.gnn{k}.phi.b"] = zeros_param(1, h)
            d_prev = h
    for head in ("sel", "plc"):
        p[f"{head}.z.w"] = glorot_uniform(rng, N_STATIC_FEATURES, h)
        p[f"{head}.z.b"] = zeros_param(1, h)
        p[f"{head}.head1.w"] = glorot_uniform(rng, 4 * h, h)
        p[f"{head}.head1.b"] = zeros_param(1, h)
        p[f"{head}.head2.w"] = glorot_uniform(rng, h, 1)
        p[f"{head}.head2.b"] = zeros_param(1, 1)
    p["plc.y.w"] = glorot_uniform(rng, N_DEVICE_FEATURES, h)
    p["plc.y.b"] = zeros_param(1, h)
    return p


def param_shapes(config) -> dict[str, tuple[int, int]]:
    h = config.hidden
    out = {}
    for enc in encoder_names(config):
        d_prev = N_STATIC_FEATURES + N_DYNAMIC_COLS
        for k in range(config.k_rounds):
            out[f"{enc}.gnn{k}.psi.w"] = (2 * d_prev + 1, h)
            out[f"{enc}.gnn{k}.psi.b"] = (1, h)
            out[f"{enc}.gnn{k}.phi.w"] = (d_prev + h, h)
            out[f"{enc}.gnn{k}.phi.b"] = (1, h)
            d_prev = h
    for head in ("sel", "plc"):
        out[f"{head}.z.w"] = (N_STATIC_FEATURES, h)
        out[f"{head}.z.b"] = (1, h)
        out[f"{head}.head1.w"] = (4 * h, h)
        out[f"{head}.head1.b"] = (1, h)
        out[f"{head}.head2.w"] = (h, 1)
        out[f"{head}.head2.b"] = (1, 1)
    out["plc.y.w"] = (N_DEVICE_FEATURES, h)
    out["plc.y.b"] = (1, h)
    return out


@dataclass
class FlatLayout:
    """name -> (offset, rows, cols) in the flat float64 parameter vector."""

    entries: dict[str, tuple[int, int, int]]
    size: int

    @classmethod
    def for_config(cls, config) -> "FlatLayout":
        off = 0
        ent = {}
        for name, (r, c) in sorted(param_shapes(config).items()):
            ent[name] = (off, r, c)
            off += r * c
        return cls(ent, off)

    def flatten(self, params: Params) -> np.ndarray:
        out = np.empty(self.size, dtype=np.float64)
        for name, (off, r, c) in self.entries.items():
            a = as_array(params[name])
            if a.shape != (r, c):
                raise ValueError(f"param {name} has shape {a.shape}, expected {(r, c)}")
            out[off:off + r * c] = a.reshape(-1)
        return out

    def unflatten(self, flat: np.ndarray) -> Params:
        return {name: Param(np.array(flat[off:off + r * c]).reshape(r, c))
                for name, (off, r, c) in self.entries.items()}

    def offset(self, name: str) -> int:
        return self.entries[name][0] if name in self.entries else -1


def params_to_dict(params: Params) -> dict:
    return {"version": CHECKPOINT_VERSION,
            "tensors": {name: {"shape": list(as_array(t).shape),
                               "values": as_array(t).reshape(-1).tolist()}
                        for name, t in sorted(params.items())}}


def params_from_dict(doc: dict) -> Params:
    if doc.get("version") != CHECKPOINT_VERSION:
        raise ValueError(f"unsupported checkpoint version {doc.get('version')!r}")
    return {name: Param(np.asarray(rec["values"], dtype=np.float64).reshape(tuple(rec["shape"])))
            for name, rec in doc["tensors"].items()}


def save_params(params: Params, path: str | Path) -> None:
    Path(path).write_text(json.dumps(params_to_dict(params)) + "\n")


def load_params(path: str | Path) -> Params:
    return params_from_dict(json.loads(Path(path).read_text()))
