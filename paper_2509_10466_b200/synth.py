"""Seeded synthetic inputs for the BASELINE.json configs.

The reference measures on no public dataset for this path; BASELINE.json's configs are
synthetic, and these generators restate them with `numpy.random.default_rng(seed)`:

* C1  1x3x256^2 blurred-uniform image + one axis-aligned rectangle (10-25% area)
* C2  1x3x512^2 frames, seed per frame; 1-4 ellipses U[20,120] semi-axes plus a 15 px
      random-walk brush stroke, forced to [0.05, 0.30] by the reference's area adjuster
* C3  8 streams x 300 frames: a smooth canvas translating 2 px/frame + N(0, 0.01) noise,
      one ellipse (15-25%) jittering +-4 px/frame
* C4  1x3x1024^2, 2-6 ellipses forced to [0.30, 0.45]
* C5  batches of 512^2 frames, masks a seeded mix of rectangles, strokes and ellipse
      unions forced to [0.05, 0.45]

Images are float32 in [0,1], (3, H, W); masks are bool (H, W).  Host-side numpy only.
"""

from __future__ import annotations

import math

import numpy as np

from .masks import adjust_mask_area_bits


def _gauss_taps(sigma: float) -> np.ndarray:
    r = int(4.0 * sigma + 0.5)
    x = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (x / sigma) ** 2)
    return w / w.sum()


def blur(img: np.ndarray, sigma: float) -> np.ndarray:
    """Separable Gaussian over the last two axes, 'reflect' borders (d c b a | a b c d)."""
    w = _gauss_taps(sigma)
    r = (len(w) - 1) // 2
    out = img.astype(np.float64)
    for axis in (-2, -1):
        n = out.shape[axis]
        pad = [(0, 0)] * out.ndim
        pad[axis] = (r, r)
        p = np.pad(out, pad, mode="symmetric")
        acc = np.zeros_like(out)
        for j in range(len(w)):
            acc += w[j] * np.take(p, np.arange(j, j + n), axis=axis)
        out = acc
    return out


def smooth_image(rng: np.random.Generator, h: int, w: int, sigma: float = 4.0) -> np.ndarray:
    """U[0,1] per channel, Gaussian blur sigma=4 (mean ~0.5, std ~0.02)."""
    return blur(rng.random((3, h, w)), sigma).astype(np.float32)


def rectangle(rng, h, w, area_min=0.10, area_max=0.25) -> np.ndarray:
    frac = rng.uniform(area_min, area_max)
    aspect = rng.uniform(0.5, 2.0)
    rw = int(np.clip(round(math.sqrt(frac * w * h * aspect)), 1, w))
    rh = int(np.clip(round(frac * w * h / rw), 1, h))
    x = int(rng.integers(0, w - rw + 1))
    y = int(rng.integers(0, h - rh + 1))
    bits = np.zeros((h, w), bool)
    bits[y:y + rh, x:x + rw] = True
    return bits


def ellipse(h, w, cy, cx, ay, ax) -> np.ndarray:
    yy, xx = np.mgrid[0:h, 0:w]
    return ((yy - cy) / ay) ** 2 + ((xx - cx) / ax) ** 2 <= 1.0


def ellipses(rng, h, w, n_min, n_max, semi=(20.0, 120.0)) -> np.ndarray:
    bits = np.zeros((h, w), bool)
    for _ in range(int(rng.integers(n_min, n_max + 1))):
        ay, ax = rng.uniform(semi[0], semi[1], size=2)
        cy, cx = rng.uniform(0, h), rng.uniform(0, w)
        bits |= ellipse(h, w, cy, cx, ay, ax)
    return bits


def thick_polyline(h, w, pts, width) -> np.ndarray:
    """Pixels whose centre lies within width/2 of any segment of the polyline."""
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    bits = np.zeros((h, w), bool)
    r2 = (width / 2.0) ** 2
    for (y0, x0), (y1, x1) in zip(pts[:-1], pts[1:]):
        dy, dx = y1 - y0, x1 - x0
        L2 = dy * dy + dx * dx
        t = np.zeros_like(yy) if L2 == 0 else \
            np.clip(((yy - y0) * dy + (xx - x0) * dx) / L2, 0.0, 1.0)
        bits |= (yy - (y0 + t * dy)) ** 2 + (xx - (x0 + t * dx)) ** 2 <= r2
    return bits


def brush_stroke(rng, h, w, width=15.0) -> np.ndarray:
    """Random-walk polyline: 4-9 steps of 20-60 px with a drifting heading."""
    n = int(rng.integers(4, 10))
    y, x = rng.uniform(0, h), rng.uniform(0, w)
    heading = rng.uniform(0, 2 * math.pi)
    pts = [(y, x)]
    for _ in range(n):
        heading += rng.normal(0.0, 0.8)
        step = rng.uniform(20, 60)
        y = float(np.clip(y + step * math.sin(heading), 0, h - 1))
        x = float(np.clip(x + step * math.cos(heading), 0, w - 1))
        pts.append((y, x))
    return thick_polyline(h, w, pts, width)


# --------------------------------------------------------------------------- configs
def c1_frame(seed: int = 0, size: int = 256):
    """C1: image then rectangle from the same stream."""
    rng = np.random.default_rng(seed)
    img = smooth_image(rng, size, size)
    return img, rectangle(rng, size, size, 0.10, 0.25)


def c2_frame(seed: int, size: int = 512):
    """C2: one real-time frame per seed."""
    rng = np.random.default_rng(seed)
    img = smooth_image(rng, size, size)
    bits = ellipses(rng, size, size, 1, 4) | brush_stroke(rng, size, size, 15.0)
    return img, adjust_mask_area_bits(bits, 0.05, 0.30)


def c4_frame(seed: int = 0, size: int = 1024):
    rng = np.random.default_rng(seed)
    img = smooth_image(rng, size, size)
    bits = ellipses(rng, size, size, 2, 6, semi=(40.0, 240.0))
    return img, adjust_mask_area_bits(bits, 0.30, 0.45)


def c5_frame(seed: int, size: int = 512):
    rng = np.random.default_rng(seed)
    img = smooth_image(rng, size, size)
    kind = int(rng.integers(0, 3))
    if kind == 0:
        bits = rectangle(rng, size, size, 0.05, 0.45)
    elif kind == 1:
        bits = np.zeros((size, size), bool)
        for _ in range(int(rng.integers(1, 6))):
            bits |= brush_stroke(rng, size, size, float(rng.integers(5, 21)))
    else:
        bits = ellipses(rng, size, size, 1, 4)
    return img, adjust_mask_area_bits(bits, 0.05, 0.45)


class C3Stream:
    """C3: one stream of frames over a translating smooth canvas."""

    def __init__(self, stream: int, size: int = 512, frames: int = 300):
        rng = np.random.default_rng(1000 + stream)
        self.size = size
        self.frames = frames
        span = size + 2 * frames + 16
        self.canvas = blur(rng.random((3, size + 16, span)), 8.0).astype(np.float32)
        frac = rng.uniform(0.15, 0.25)
        aspect = rng.uniform(0.7, 1.4)
        area = frac * size * size
        self.ay = math.sqrt(area / math.pi / aspect)
        self.ax = self.ay * aspect
        self.cy = rng.uniform(self.ay, size - self.ay)
        self.cx = rng.uniform(self.ax, size - self.ax)
        self.seed = 1000 + stream

    def frame(self, t: int):
        rng = np.random.default_rng([self.seed, t])
        x0 = 2 * t
        img = self.canvas[:, 8:8 + self.size, x0:x0 + self.size]
        img = np.clip(img + rng.normal(0.0, 0.01, img.shape), 0.0, 1.0).astype(np.float32)
        jy, jx = rng.integers(-4, 5, size=2)
        bits = ellipse(self.size, self.size, self.cy + jy, self.cx + jx, self.ay, self.ax)
        return img, bits


def frame_pool(config: str, n: int, size: int | None = None):
    """n (image, mask) pairs of a config, stacked: (n,3,H,W) f32, (n,H,W) bool."""
    gen = {"C1": lambda s: c1_frame(s, size or 256),
           "C2": lambda s: c2_frame(s, size or 512),
           "C4": lambda s: c4_frame(s, size or 1024),
           "C5": lambda s: c5_frame(s, size or 512)}[config]
    imgs, masks = zip(*(gen(s) for s in range(n)))
    return np.stack(imgs), np.stack(masks)
