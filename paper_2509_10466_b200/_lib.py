"""ctypes binding of libdrb200.so (the C-ABI declared in include/dr_b200.h).

The library is loaded from the package's in-tree `_build/` directory.  There is no
fallback: if the library or a CUDA device is missing every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import ConfigError, DeviceError, EngineNumericError, InputError

LIB_PATH = Path(os.environ.get("DR_B200_LIB", Path(__file__).resolve().parent / "_build" /
                               "libdrb200.so"))

DR_OK, DR_ERR_CONFIG, DR_ERR_INPUT, DR_ERR_NUMERIC, DR_ERR_CUDA = 0, 1, 2, 3, 4
DR_FLAG_NONFINITE, DR_FLAG_UNREDACTED = 1, 2


class DrConfig(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("patch", ctypes.c_int32), ("channels", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("heads", ctypes.c_int32),
                ("temporal_groups", ctypes.c_int32), ("n_blocks", ctypes.c_int32),
                ("blocks", ctypes.c_char * 16), ("mask_dilate", ctypes.c_int32),
                ("mask_feather_sigma", ctypes.c_float),
                ("mask_aware_attention", ctypes.c_int32)]


class DrFrameIO(ctypes.Structure):
    _fields_ = [("frames", ctypes.c_int32), ("rgb_f32", ctypes.c_void_p),
                ("rgb_u8", ctypes.c_void_p), ("mask_m0", ctypes.c_void_p),
                ("slot0", ctypes.c_void_p), ("slot1", ctypes.c_void_p),
                ("slot_batched", ctypes.c_int32), ("new_slot", ctypes.c_void_p),
                ("out_f32", ctypes.c_void_p), ("out_u8", ctypes.c_void_p),
                ("fill", ctypes.c_void_p), ("dilated", ctypes.c_void_p),
                ("alpha", ctypes.c_void_p), ("token_valid", ctypes.c_void_p),
                ("flags", ctypes.c_void_p), ("slot_kv_reuse", ctypes.c_int32)]


# symbol -> (restype, argtypes); the export test checks this against include/dr_b200.h
SIGNATURES = {
    "dr_create": (ctypes.c_int, [ctypes.POINTER(DrConfig), ctypes.POINTER(ctypes.c_void_p),
                                 ctypes.POINTER(ctypes.c_int64), ctypes.c_int32,
                                 ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
    "dr_destroy": (None, [ctypes.c_void_p]),
    "dr_last_error": (ctypes.c_char_p, []),
    "dr_version": (ctypes.c_int32, []),
    "dr_forward": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(DrFrameIO), ctypes.c_void_p]),
    "dr_mask_stage": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_int32, ctypes.c_int32, ctypes.c_float,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p]),
    "dr_inpaint_u8_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "dr_inpaint_u8_host_mem": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "dr_reset_memory": (ctypes.c_int, [ctypes.c_void_p]),
    "dr_kernels_per_forward": (ctypes.c_int32, [ctypes.c_void_p]),
    "dr_token_tile_rows": (ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32]),
    "dr_host_d2h_bytes": (ctypes.c_int64, [ctypes.c_void_p]),
    "dr_op_conv3x3": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p]),
    "dr_profile": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "dr_display_composite": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]),
    "dr_merge_redact": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "dr_pack_pointcloud": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_double, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    "dr_profile_read": (ctypes.c_int32, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float),
                                         ctypes.POINTER(ctypes.c_int32), ctypes.c_int32]),
}

STAGE_NAMES = {0: "mask_stage", 1: "slot_kv", 2: "embed_qkv", 3: "attn_spatial",
               4: "attn_temporal", 5: "mlp_qkv", 6: "vec2patch", 7: "decode0",
               8: "decode2_composite", 9: "decoder_fused", 10: "seam_fixup", 11: "dec_border"}

_lib = None


def load():
    """Load and type the library (no CUDA calls happen at load time)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == DR_OK:
        return
    msg = (load().dr_last_error() or b"").decode(errors="replace")
    exc = {DR_ERR_CONFIG: ConfigError, DR_ERR_INPUT: InputError,
           DR_ERR_NUMERIC: EngineNumericError}.get(rc, DeviceError)
    raise exc(msg)


def make_config(cfg) -> DrConfig:
    c = DrConfig()
    c.width, c.height, c.patch = cfg.width, cfg.height, cfg.patch
    c.channels, c.kernel, c.heads = cfg.channels, cfg.kernel, cfg.heads
    c.temporal_groups = cfg.temporal_groups
    if len(cfg.blocks) > 16:
        raise ConfigError("at most 16 blocks")
    c.n_blocks = len(cfg.blocks)
    c.blocks = "".join(cfg.blocks).encode()
    c.mask_dilate = int(cfg.mask_dilate)
    c.mask_feather_sigma = float(cfg.mask_feather_sigma)
    c.mask_aware_attention = int(bool(cfg.mask_aware_attention))
    return c


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("the B200 engine needs a CUDA device (there is no CPU fallback)")
    return torch


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def mask_stage(m0, radius: int, sigma: float, patch: int):
    """Device mask stage on a CUDA (B, H, W) or (H, W) mask (see masks.py).

    Returns (m1 u8, alpha f32, token_valid u8 or None when patch does not tile)."""
    torch = require_cuda()
    if m0.dim() == 2:
        m0 = m0[None]
    if not m0.is_cuda:
        raise DeviceError("mask must be a CUDA tensor")
    b, h, w = m0.shape
    m0 = m0.to(torch.uint8).contiguous()
    m1 = torch.empty_like(m0)
    alpha = torch.empty(m0.shape, dtype=torch.float32, device=m0.device)
    tv = None
    if patch in (4, 8) and h % patch == 0 and w % patch == 0:
        tv = torch.empty((b, (h // patch) * (w // patch)), dtype=torch.uint8, device=m0.device)
    check(load().dr_mask_stage(b, h, w, patch, int(radius), float(sigma), m0.data_ptr(),
                               m1.data_ptr(), alpha.data_ptr(), ptr(tv),
                               stream_handle(m0.device)))
    return m1, alpha, tv
