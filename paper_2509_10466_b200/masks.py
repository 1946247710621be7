"""Privacy-mask utilities: the reference's host types plus the device mask stage.

Host (numpy), same semantics as the reference `pkg/src/dimreal/masks.py`:
`BinaryMask` (:20-125), `redact` (:145-154), `adjust_mask_area` with the 3x3-cross
dilation/erosion (:17, :182-201).

Device (CUDA, via the C-ABI `dr_mask_stage`): `dilate_mask`, `feather_mask`,
`token_mask` run the SMEM stencil kernel of `csrc/mask_kernels.cu` on CUDA tensors.
There is no CPU fallback: without the extension or a GPU they raise.
"""

from __future__ import annotations

import dataclasses

import numpy as np

from .errors import DegenerateMaskError, InputError


class BinaryMask:
    """Per-pixel boolean redaction region (masks.py:20-125)."""

    __slots__ = ("bits", "_bbox")

    def __init__(self, bits):
        bits = np.asarray(bits)
        if bits.dtype != np.bool_:
            bits = bits.astype(bool)
        if bits.ndim != 2:
            raise InputError("mask must be a 2-D raster")
        self.bits = bits
        self._bbox = None

    @classmethod
    def empty(cls, width: int, height: int) -> "BinaryMask":
        return cls(np.zeros((height, width), dtype=bool))

    @classmethod
    def full(cls, width: int, height: int) -> "BinaryMask":
        return cls(np.ones((height, width), dtype=bool))

    @property
    def width(self) -> int:
        return self.bits.shape[1]

    @property
    def height(self) -> int:
        return self.bits.shape[0]

    def area(self) -> int:
        return int(np.count_nonzero(self.bits))

    def area_fraction(self) -> float:
        return self.area() / self.bits.size

    def is_empty(self) -> bool:
        return not self.bits.any()

    def union(self, other: "BinaryMask") -> "BinaryMask":
        if other.bits.shape != self.bits.shape:
            raise InputError("mask dimensions differ")
        return BinaryMask(self.bits | other.bits)

    def intersection(self, other: "BinaryMask") -> "BinaryMask":
        if other.bits.shape != self.bits.shape:
            raise InputError("mask dimensions differ")
        return BinaryMask(self.bits & other.bits)

    def tight_bbox(self) -> tuple[int, int, int, int]:
        """(x, y, w, h) of the true pixels."""
        if self._bbox is None:
            ys = np.flatnonzero(self.bits.any(axis=1))
            if ys.size == 0:
                raise InputError("empty mask has no bounding box")
            xs = np.flatnonzero(self.bits.any(axis=0))
            self._bbox = (int(xs[0]), int(ys[0]),
                          int(xs[-1] - xs[0] + 1), int(ys[-1] - ys[0] + 1))
        return self._bbox

    def __eq__(self, other) -> bool:
        return isinstance(other, BinaryMask) and self.bits.shape == other.bits.shape \
            and bool(np.array_equal(self.bits, other.bits))

    def __repr__(self) -> str:
        return f"BinaryMask({self.width}x{self.height}, area={self.area()})"


def redact(frame, mask: BinaryMask):
    """Zero the rgb pixels inside the mask (masks.py:145-154).  ``frame`` is a
    dataclass with an ``rgb`` (H, W, 3) array (the reference's FrameRGBD) or a bare
    (H, W, 3) array."""
    rgb_in = frame if isinstance(frame, np.ndarray) else frame.rgb
    if mask.bits.shape != rgb_in.shape[:2]:
        raise InputError("mask dimensions do not match frame")
    rgb = rgb_in.copy()
    if not mask.is_empty():
        x, y, w, h = mask.tight_bbox()
        rgb[y:y + h, x:x + w][mask.bits[y:y + h, x:x + w]] = 0
    rgb.flags.writeable = False
    if isinstance(frame, np.ndarray):
        return rgb
    return dataclasses.replace(frame, rgb=rgb)


def _cross_dilate(bits):
    out = bits.copy()
    out[1:, :] |= bits[:-1, :]
    out[:-1, :] |= bits[1:, :]
    out[:, 1:] |= bits[:, :-1]
    out[:, :-1] |= bits[:, 1:]
    return out


def _cross_erode(bits):
    out = bits.copy()
    out[1:, :] &= bits[:-1, :]
    out[:-1, :] &= bits[1:, :]
    out[:, 1:] &= bits[:, :-1]
    out[:, :-1] &= bits[:, 1:]
    out[0, :] = False
    out[-1, :] = False
    out[:, 0] = False
    out[:, -1] = False
    return out


def adjust_mask_area_bits(bits: np.ndarray, area_min: float, area_max: float) -> np.ndarray:
    """masks.py:182-201 on a bool array: grow by the cross while below ``area_min``
    (stop when saturated), then erode (off-frame = empty) while above ``area_max``."""
    bits = np.asarray(bits, bool)
    if not bits.any():
        raise DegenerateMaskError("cannot adjust an empty mask")
    total = bits.size
    while np.count_nonzero(bits) / total < area_min:
        grown = _cross_dilate(bits)
        if np.count_nonzero(grown) == np.count_nonzero(bits):
            break
        bits = grown
    while np.count_nonzero(bits) / total > area_max:
        bits = _cross_erode(bits)
        if not bits.any():
            raise DegenerateMaskError("mask eroded to empty before reaching bounds")
    return bits


def adjust_mask_area(mask: BinaryMask, area_min: float, area_max: float) -> BinaryMask:
    return BinaryMask(adjust_mask_area_bits(mask.bits, area_min, area_max))


# ------------------------------------------------------------------ device mask stage
def mask_stage(m0, radius: int, sigma: float, patch: int):
    """Run the fused device mask stage on a CUDA uint8/bool tensor (B, H, W).

    Returns (m1 u8 (B,H,W), alpha f32 (B,H,W), token_valid u8 (B,T))."""
    from . import _lib
    return _lib.mask_stage(m0, radius, sigma, patch)


def dilate_mask(m0, radius: int):
    """m1 = m0 dilated ``radius`` times by the 3x3 cross (L1 ball), on device."""
    return mask_stage(m0, radius, 0.0, 1)[0]


def feather_mask(m1, sigma: float):
    """alpha = max(m1, G_sigma(m1)) (scipy gaussian_filter semantics), on device."""
    return mask_stage(m1, 0, sigma, 1)[1]


def token_mask(m1, patch: int):
    """valid[t] = any pixel of patch t outside m1, on device."""
    return mask_stage(m1, 0, 0.0, patch)[2]
