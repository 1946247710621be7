"""The reference's own CPU implementation of the hot path, for bench.py's reference arm.

Runs the UNMODIFIED reference package `dimreal` installed into `baseline/_ref/` by
`baseline/install_ref.sh` (pip --target from a copy of /root/reference/pkg; git-ignored,
travels to the GPU box with the repo snapshot).  Nothing of this repository is on the
path it times:

* dilation   scipy.ndimage.binary_dilation(m0, structure=dimreal.masks._CROSS,
             iterations=r)          -- the reference's own primitive (masks.py:17, :193)
* feather    scipy.ndimage.gaussian_filter(m1, sigma, mode='nearest', truncate=4),
             alpha = max(m1, G)     -- SURVEY §8(a) A3
* network    dimreal.inpaint.dstt.DsttEngine(DsttConfig(W, H, temporal_groups=4),
             seed=0).model, forward under torch.no_grad on the frame redacted inside m1
             with m1 as the mask channel (dstt.py:256-268, masks.py:145-154)
* composite  out = alpha*fill + (1-alpha)*frame in fp32

Memory is carried across frames for the streaming configs (dstt.py:309-311,
memory.py:40-45).  torch intra-op threads = the host cores given.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"


def available() -> str | None:
    """None when the installed reference imports, else the reason it does not."""
    if not (REF_DIR / "dimreal").is_dir():
        return f"{REF_DIR} missing (run baseline/install_ref.sh)"
    try:
        _import()
    except Exception as e:  # pragma: no cover - depends on the install
        return f"dimreal import failed: {type(e).__name__}: {e}"
    return None


def _import():
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_dimreal")
    import dimreal.masks as masks
    from dimreal.inpaint import dstt
    return masks, dstt


class ReferencePath:
    """One frame (or a batch of independent frames) through the reference's CPU path."""

    def __init__(self, size: int, radius: int = 5, sigma: float = 3.0, threads: int | None = None):
        import torch
        masks, dstt = _import()
        from scipy import ndimage
        self.torch, self.ndimage, self.cross = torch, ndimage, masks._CROSS
        torch.set_num_threads(threads or os.cpu_count() or 1)
        self.cfg = dstt.DsttConfig(width=size, height=size, temporal_groups=4)
        self.model = dstt.DsttEngine(self.cfg, seed=0).model
        self.radius, self.sigma = radius, sigma
        zero = torch.zeros(1, self.cfg.tokens, self.cfg.channels)
        self.slots = (zero, zero)
        self.threads = torch.get_num_threads()

    def masks(self, m0: np.ndarray):
        nd = self.ndimage
        m1 = nd.binary_dilation(m0, structure=self.cross, iterations=self.radius) \
            if self.radius > 0 else m0.astype(bool)
        f = m1.astype(np.float32)
        alpha = np.maximum(f, nd.gaussian_filter(f, self.sigma, mode="nearest", truncate=4.0)) \
            if self.sigma > 0 else f
        return m1, alpha

    def step(self, img: np.ndarray, m0: np.ndarray, carried: bool) -> np.ndarray:
        """img (3,H,W) f32 in [0,1], m0 (H,W) bool -> composite (3,H,W) f32."""
        torch = self.torch
        m1, alpha = self.masks(m0)
        rgb = np.where(m1[None], np.float32(0.0), img).astype(np.float32)
        x = torch.from_numpy(rgb)[None]
        m = torch.from_numpy(m1.astype(np.float32))[None, None]
        with torch.no_grad():
            fill, new_slot = self.model(x, m, self.slots)
        if carried:
            self.slots = (self.slots[1], new_slot)
        fill = fill[0].numpy()
        a = alpha[None]
        return (a * fill + (np.float32(1.0) - a) * img).astype(np.float32)


def time_frames(path: ReferencePath, frames, carried: bool, warmup: int, steps: int):
    """Per-frame seconds of `steps` timed frames after `warmup` untimed ones, cycling
    through `frames` [(img, m0), ...]."""
    times = []
    for k in range(warmup + steps):
        img, m0 = frames[k % len(frames)]
        t0 = time.perf_counter()
        path.step(img, m0, carried)
        dt = time.perf_counter() - t0
        if k >= warmup:
            times.append(dt)
    return times
