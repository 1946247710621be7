"""B200-native masked-inpainting hot path of arXiv 2509.10466 (`dimreal` drop-in).

Public names follow the reference package (`pkg/src/dimreal/__init__.py:3-18`,
`inpaint/__init__.py:1-22`) for the path this package replaces:

    DsttConfig, DsttEngine, InpaintEngine, EngineResult, InpaintMemory, memory_push,
    load_weights, save_weights, BinaryMask, redact, adjust_mask_area,
    dilate_mask, feather_mask, token_mask (device mask stage, new),
    BatchStreamer (overlapped pinned-host batches, new)

The compute path is `libdrb200.so` (hand-written sm_100a CUDA behind a C-ABI, see
`include/dr_b200.h`); there is no CPU fallback.
"""

from .config import DsttConfig
from .errors import (ConfigError, DegenerateMaskError, DeviceError, EngineNumericError,
                     InputError)
from .masks import (BinaryMask, adjust_mask_area, dilate_mask, feather_mask, redact,
                    token_mask)
from .memory import InpaintMemory, memory_push
from .weights import load_weights, save_weights

__all__ = [
    "BatchStreamer", "BinaryMask", "ConfigError", "DegenerateMaskError", "DeviceError", "DsttConfig",
    "DsttEngine", "EngineNumericError", "EngineResult", "InpaintEngine", "InpaintMemory",
    "InputError", "adjust_mask_area", "dilate_mask", "feather_mask", "load_weights",
    "memory_push", "redact", "save_weights", "token_mask",
]


def __getattr__(name):
    if name in ("DsttEngine", "InpaintEngine", "EngineResult"):
        from . import engine
        return getattr(engine, name)
    if name == "BatchStreamer":
        from .streaming import BatchStreamer
        return BatchStreamer
    raise AttributeError(name)
