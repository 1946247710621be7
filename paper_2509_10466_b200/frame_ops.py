"""Frame byte kernels either side of the network, on the device.

Host mirror of the reference entry points (under /root/reference/pkg/src/dimreal):

* `upscale2x(raster)`                          pipeline.upscale2x (pipeline.py:120-131)
* `display_output(original, inpainted, mask, engine_failed)`
                                               Pipeline.step's display stage
                                               (pipeline.py:307-314) with
                                               _composite_upscaled (pipeline.py:203-222)
* `merge_private_masks(tracks, width, height)` masks.merge_private_masks (masks.py:128-142)
* `merge_and_redact(masks, private, rgb)`      merge_private_masks + redact (masks.py:145-154)
* `transplant_pointcloud(rgb, depth, intrinsics, frame_id)`
                                               pipeline.transplant_pointcloud
                                               (pipeline.py:147-157, _kernels.py:49-93)

Arguments may be numpy arrays (copied to the current CUDA device; results come back as
numpy, like the reference) or CUDA tensors (results stay on the device).  Errors follow
the reference: wrong dtype / shape -> InputError.  There is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InputError


def _dev(x, dtype):
    """(tensor on device, was_numpy)."""
    torch = _lib.require_cuda()
    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x)).cuda(), True
    if not x.is_cuda:
        return x.contiguous().cuda(), True
    return x.contiguous(), False


def _is_u8(x) -> bool:
    if isinstance(x, np.ndarray):
        return x.dtype == np.uint8
    import torch
    return x.dtype == torch.uint8


def _out(t, host: bool):
    return t.cpu().numpy() if host else t


def upscale2x(raster):
    """Bilinear 2x of a uint8 (H, W) or (H, W, 3) raster, half-pixel centres, round half up:
    out[2y+ky, 2x+kx] = (9a + 3a_y2 + 3a_x2 + a_y2x2 + 8) >> 4 (_kernels.py:13-46)."""
    if not _is_u8(raster):
        raise InputError("upscale2x expects a uint8 raster")
    return display_output(raster, None, None)


def display_output(original, inpainted, mask, engine_failed: bool = False):
    """The privatized display frame of Pipeline.step (pipeline.py:307-314): upscale2x of the
    original, with the nearest-upscaled mask region taken from upscale2x(inpainted), or
    zeroed when ``engine_failed``.  One fused kernel (no separate up_original pass)."""
    torch = _lib.require_cuda()
    if not _is_u8(original) or (inpainted is not None and not _is_u8(inpainted)):
        raise InputError("display composite expects uint8 rasters")
    o, host = _dev(original, np.uint8)
    squeeze = o.dim() == 2
    if squeeze:
        o = o[..., None]
    if o.dim() != 3 or o.shape[2] not in (1, 3):
        raise InputError("raster must be (H, W) or (H, W, 3)")
    h, w, c = o.shape
    inp = None
    if inpainted is not None:
        inp, _ = _dev(inpainted, np.uint8)
        if inp.dim() == 2:
            inp = inp[..., None]
        if tuple(inp.shape) != (h, w, c):
            raise InputError("rgb and inpainted dimensions differ")
    m = None
    if mask is not None:
        bits = getattr(mask, "bits", mask)
        m, _ = _dev(bits if not isinstance(bits, np.ndarray) else bits.astype(np.uint8),
                    np.uint8)
        m = m.to(torch.uint8)
        if tuple(m.shape) != (h, w):
            raise InputError("mask dimensions do not match frame")
    out = torch.empty((2 * h, 2 * w, c), dtype=torch.uint8, device=o.device)
    _lib.check(_lib.load().dr_display_composite(
        h, w, c, o.data_ptr(), _lib.ptr(inp), _lib.ptr(m), int(bool(engine_failed)),
        out.data_ptr(), _lib.stream_handle(o.device)))
    if squeeze:
        out = out[..., 0]
    return _out(out, host)


def merge_and_redact(masks, private, rgb=None):
    """Union of the masks whose ``private`` flag is set (merge_private_masks) and, if
    ``rgb`` is given, the rgb raster zeroed inside the union (redact).  Returns
    (merged u8 (H, W), redacted (H, W, 3) or None)."""
    torch = _lib.require_cuda()
    mk, host = _dev(np.asarray(masks, np.uint8) if isinstance(masks, np.ndarray) else masks,
                    np.uint8)
    mk = mk.to(torch.uint8)
    if mk.dim() == 2:
        mk = mk[None]
    n, h, w = mk.shape
    pf, _ = _dev(np.asarray(private, np.uint8) if not hasattr(private, "is_cuda") else private,
                 np.uint8)
    pf = pf.to(torch.uint8).reshape(-1)
    if pf.numel() != n:
        raise InputError("one private flag per mask is required")
    merged = torch.empty((h, w), dtype=torch.uint8, device=mk.device)
    red = src = None
    if rgb is not None:
        if not _is_u8(rgb):
            raise InputError("rgb must be uint8")
        src, _ = _dev(rgb, np.uint8)
        if tuple(src.shape) != (h, w, 3):
            raise InputError("mask dimensions do not match frame")
        red = torch.empty_like(src)
    _lib.check(_lib.load().dr_merge_redact(n, h, w, mk.data_ptr(), pf.data_ptr(), _lib.ptr(src),
                                           merged.data_ptr(), _lib.ptr(red),
                                           _lib.stream_handle(mk.device)))
    return _out(merged, host), (None if red is None else _out(red, host))


def merge_private_masks(tracks, width: int, height: int):
    """masks.merge_private_masks (masks.py:128-142) on the device: ``tracks`` carry a
    ``state`` (PRIVATE by name) and ``latest.mask.bits``.  Returns a BinaryMask."""
    from .masks import BinaryMask
    bits, flags = [], []
    for t in tracks:
        b = np.asarray(t.latest.mask.bits, bool)
        if b.shape != (height, width):
            raise InputError(f"track {t.id} mask is {b.shape[1]}x{b.shape[0]}, "
                             f"frame is {width}x{height}")
        bits.append(b)
        flags.append(getattr(t.state, "name", t.state) == "PRIVATE")
    if not bits:
        return BinaryMask.empty(width, height)
    merged, _ = merge_and_redact(np.stack(bits).astype(np.uint8), np.array(flags, np.uint8))
    return BinaryMask(np.asarray(merged, bool))


@dataclass(frozen=True)
class PointCloud:
    """pipeline.PointCloud (pipeline.py:134-144)."""
    xyz: object           # (N, 3) float32
    rgb: object           # (N, 3) uint8
    frame_id: int

    def __len__(self) -> int:
        return int(self.xyz.shape[0])


def transplant_pointcloud(rgb, depth, intrinsics, frame_id: int = -1) -> PointCloud:
    """Back-project every valid-depth pixel (row-major), colored from the inpainted raster
    (pipeline.transplant_pointcloud, pipeline.py:147-157; bit-identical to the numba
    pack_pointcloud, _kernels.py:49-93)."""
    torch = _lib.require_cuda()
    r, host = _dev(rgb, np.uint8)
    d, _ = _dev(np.asarray(depth, np.float32) if isinstance(depth, np.ndarray) else depth,
                np.float32)
    d = d.to(torch.float32)
    if tuple(r.shape[:2]) != tuple(d.shape):
        raise InputError("rgb and depth dimensions differ")
    h, w = d.shape
    dev = d.device
    xyz = torch.empty((h * w, 3), dtype=torch.float32, device=dev)
    col = torch.empty((h * w, 3), dtype=torch.uint8, device=dev)
    scratch = torch.empty(max(h, 1) + 1, dtype=torch.int32, device=dev)
    _lib.check(_lib.load().dr_pack_pointcloud(
        h, w, d.data_ptr(), r.data_ptr(), float(intrinsics.fx), float(intrinsics.fy),
        float(intrinsics.cx), float(intrinsics.cy), scratch.data_ptr(), xyz.data_ptr(),
        col.data_ptr(), scratch[h:].data_ptr(), _lib.stream_handle(dev)))
    n = int(scratch[h].item())
    return PointCloud(xyz=_out(xyz[:n], host), rgb=_out(col[:n], host), frame_id=frame_id)
