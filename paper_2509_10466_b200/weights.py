"""DRWT flat weight files and the seeded random init.

File format (all integers little-endian), identical to the reference
`pkg/src/dimreal/inpaint/weights.py:1-13`:

    magic "DRWT" | version u8 = 1 | count u32 | count x (ndim u8, ndim x u32 dims)
    | float32 data of every tensor in table order

Tensors are positional, in the reference `DsttModel.state_dict()` order, which
`parameter_specs` restates from `dstt.py:231-244` and `:102-133`.
"""

from __future__ import annotations

import math
import struct
from pathlib import Path

import numpy as np

from .config import DsttConfig
from .errors import ConfigError

MAGIC = b"DRWT"
VERSION = 1


def save_weights(arrays, path) -> None:
    arrays = [np.asarray(a, dtype=np.float32) for a in arrays]
    head = [MAGIC, struct.pack("<BI", VERSION, len(arrays))]
    for arr in arrays:
        head.append(struct.pack("<B", arr.ndim))
        head.append(struct.pack(f"<{arr.ndim}I", *arr.shape))
    body = [np.ascontiguousarray(arr).astype("<f4").tobytes() for arr in arrays]
    Path(path).write_bytes(b"".join(head + body))


def load_weights(path) -> list[np.ndarray]:
    data = Path(path).read_bytes()
    if len(data) < 9:
        raise ConfigError("weights file truncated before header")
    if data[:4] != MAGIC:
        raise ConfigError(f"bad magic {data[:4]!r} in weights file")
    version, count = struct.unpack_from("<BI", data, 4)
    if version != VERSION:
        raise ConfigError(f"unsupported weights version {version}")
    pos = 9
    shapes = []
    for _ in range(count):
        if pos + 1 > len(data):
            raise ConfigError("weights file truncated in dims table")
        (ndim,) = struct.unpack_from("<B", data, pos)
        pos += 1
        if pos + 4 * ndim > len(data):
            raise ConfigError("weights file truncated in dims table")
        shapes.append(struct.unpack_from(f"<{ndim}I", data, pos))
        pos += 4 * ndim
    out = []
    for shape in shapes:
        n = int(np.prod(shape)) if shape else 1
        end = pos + 4 * n
        if end > len(data):
            raise ConfigError("weights file truncated in data section")
        out.append(np.frombuffer(data, dtype="<f4", count=n, offset=pos)
                   .reshape(shape).astype(np.float32))
        pos = end
    if pos != len(data):
        raise ConfigError("trailing bytes after weights data")
    return out


def parameter_specs(cfg: DsttConfig) -> list[tuple[str, tuple[int, ...]]]:
    """(name, shape) of every tensor in `DsttModel.state_dict()` order."""
    c, p, k = cfg.channels, cfg.patch, cfg.kernel
    specs = [("embed.weight", (c, 4, p, p)), ("embed.bias", (c,))]
    for i, _kind in enumerate(cfg.blocks):
        b = f"blocks.{i}."
        specs += [(b + "norm1.weight", (c,)), (b + "norm1.bias", (c,))]
        for proj in ("q_proj", "k_proj", "v_proj", "out_proj"):
            specs += [(b + f"attn.{proj}.weight", (c, c)), (b + f"attn.{proj}.bias", (c,))]
        specs += [(b + "norm2.weight", (c,)), (b + "norm2.bias", (c,)),
                  (b + "ffn.net.0.weight", (2 * c, c)), (b + "ffn.net.0.bias", (2 * c,)),
                  (b + "ffn.net.2.weight", (c, 2 * c)), (b + "ffn.net.2.bias", (c,))]
    specs += [("vec2patch.deconv.weight", (c, c, k, k)), ("vec2patch.deconv.bias", (c,)),
              ("decode.0.weight", (c, c, 3, 3)), ("decode.0.bias", (c,)),
              ("decode.2.weight", (3, c, 3, 3)), ("decode.2.bias", (3,))]
    return specs


def seed_parameters(cfg: DsttConfig, seed: int) -> list[np.ndarray]:
    """The reference's seeded init (`dstt.py:271-281`): one CPU torch Generator seeded
    with ``seed``; >=2-D params He-normal randn * sqrt(2/prod(shape[1:])) in parameter
    order; 1-D ``*weight`` (LayerNorm) = 1; every bias = 0.  Host-side, runs once."""
    import torch

    gen = torch.Generator().manual_seed(seed)
    out = []
    for name, shape in parameter_specs(cfg):
        if len(shape) >= 2:
            fan_in = int(np.prod(shape[1:]))
            t = torch.randn(shape, generator=gen) * math.sqrt(2.0 / fan_in)
            out.append(t.numpy().astype(np.float32))
        elif name.endswith("weight"):
            out.append(np.ones(shape, np.float32))
        else:
            out.append(np.zeros(shape, np.float32))
    return out


def check_shapes(cfg: DsttConfig, arrays) -> list[np.ndarray]:
    """Positional shape check with the reference's messages (`dstt.py:332-341`)."""
    specs = parameter_specs(cfg)
    if len(arrays) != len(specs):
        raise ConfigError(f"weights file has {len(arrays)} tensors, model needs {len(specs)}")
    out = []
    for (name, shape), arr in zip(specs, arrays):
        arr = np.asarray(arr, dtype=np.float32)
        if tuple(arr.shape) != tuple(shape):
            raise ConfigError(f"tensor {name}: file shape {arr.shape} != model shape {shape}")
        out.append(np.ascontiguousarray(arr))
    return out
