"""CPU ORACLE for the masked-inpainting hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl
reference` legs may import this module, and only as the checker or the timed CPU
reference.  The product path (`paper_2509_10466_b200`) never imports it and fails loudly
when its CUDA extension is missing.

This is a numpy restatement of the reference package `dimreal` (`/root/reference/pkg`,
read-only, not shipped).  Every function cites the reference file:line it follows.  The
reference's arithmetic lives in PyTorch CPU aten ops (torch unpinned, 2.11.0 installed)
and scipy.ndimage (unpinned, 1.18.1 installed); their published semantics are restated
here in plain numpy (scipy.special.erf for the exact-erf GELU).

Pinned: `tests/golden/*.npz` hold outputs of the reference itself, generated in the build
container by `tests/golden/make_golden.py` (committed); `tests/test_oracle.py` checks this
module against them (forward within 1e-4, masks bit-exact, feather within 1e-6).

New stages with no reference implementation are
*defined* here from reference primitives; with r=0, sigma=0, mask-aware off they reduce
to the unmodified reference.
"""

from __future__ import annotations

import math

import numpy as np

try:  # exact erf for nn.GELU(approximate='none'); scipy is a reference dependency
    from scipy.special import erf as _erf
except Exception:  # pragma: no cover - scipy is in the image
    _erf = np.vectorize(math.erf, otypes=[np.float64])

F32 = np.float32


# ----------------------------------------------------------------------------------
# A2  binary dilation of the privacy mask
# ----------------------------------------------------------------------------------
def cross_dilate_once(bits: np.ndarray) -> np.ndarray:
    """One `ndimage.binary_dilation(bits, structure=_CROSS)` (masks.py:17, :193):
    the 3x3 cross, pixels outside the frame count as 0.  bits: (..., H, W) bool."""
    out = bits.copy()
    out[..., 1:, :] |= bits[..., :-1, :]
    out[..., :-1, :] |= bits[..., 1:, :]
    out[..., :, 1:] |= bits[..., :, :-1]
    out[..., :, :-1] |= bits[..., :, 1:]
    return out


def cross_erode_once(bits: np.ndarray) -> np.ndarray:
    """`ndimage.binary_erosion(bits, structure=_CROSS)` (masks.py:198); off-frame = 0."""
    out = bits.copy()
    up = np.zeros_like(bits)
    up[..., 1:, :] = bits[..., :-1, :]
    dn = np.zeros_like(bits)
    dn[..., :-1, :] = bits[..., 1:, :]
    lf = np.zeros_like(bits)
    lf[..., :, 1:] = bits[..., :, :-1]
    rt = np.zeros_like(bits)
    rt[..., :, :-1] = bits[..., :, 1:]
    return out & up & dn & lf & rt


def dilate_mask(m0: np.ndarray, r: int) -> np.ndarray:
    """m1 = m0 dilated r times by the 3x3 cross == the L1 ball of radius r (
    growth pinned by `tests/oracles.py:82-84` diamond_area).  (..., H, W) -> bool."""
    m = np.asarray(m0).astype(bool)
    for _ in range(int(r)):
        m = cross_dilate_once(m)
    return m


def adjust_mask_area(bits: np.ndarray, area_min: float, area_max: float) -> np.ndarray:
    """masks.py:182-201: dilate by the cross while below the lower bound (stop when
    saturated), then erode while above the upper bound."""
    if not bits.any():
        raise ValueError("cannot adjust an empty mask")
    total = bits.size
    while np.count_nonzero(bits) / total < area_min:
        grown = cross_dilate_once(bits)
        if np.count_nonzero(grown) == np.count_nonzero(bits):
            break
        bits = grown
    while np.count_nonzero(bits) / total > area_max:
        bits = cross_erode_once(bits)
        if not bits.any():
            raise ValueError("mask eroded to empty before reaching bounds")
    return bits


# ----------------------------------------------------------------------------------
# A3  feather: alpha = max(m1, G_sigma(m1)), scipy.ndimage.gaussian_filter semantics
# ----------------------------------------------------------------------------------
def gaussian_kernel1d(sigma: float, radius: int) -> np.ndarray:
    """scipy.ndimage._filters._gaussian_kernel1d (order 0), float64."""
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    phi = np.exp(-0.5 / (sigma * sigma) * x * x)
    return phi / phi.sum()


def _correlate1d_nearest(a: np.ndarray, w: np.ndarray, axis: int) -> np.ndarray:
    """scipy.ndimage.correlate1d(mode='nearest') in float64, result cast to float32
    (gaussian_filter writes each pass into a float32 output array)."""
    radius = (len(w) - 1) // 2
    a64 = a.astype(np.float64)
    n = a.shape[axis]
    idx = np.clip(np.arange(-radius, n + radius), 0, n - 1)
    padded = np.take(a64, idx, axis=axis)

    def tap(d):                       # input shifted by d along axis
        sl = [slice(None)] * a.ndim
        sl[axis] = slice(radius + d, radius + d + n)
        return padded[tuple(sl)]
    # scipy NI_Correlate1D, symmetric weights: x[0]*w[0], then the pairs from the
    # outermost inward, (x[-j] + x[+j]) * w[j] -- same order, so float64-identical.
    acc = tap(0) * w[radius]
    for jj in range(-radius, 0):
        acc = acc + (tap(jj) + tap(-jj)) * w[radius + jj]
    return acc.astype(F32)


def feather_mask(m1: np.ndarray, sigma: float) -> np.ndarray:
    """alpha = max(m1, gaussian_filter(m1.astype(f32), sigma, mode='nearest',
    truncate=4.0)), filtered over the two spatial axes, axis H first then W (scipy's
    axis order).  The max keeps alpha == 1 on m1 (so m0 never leaks).  sigma=0 -> m1."""
    m = np.asarray(m1).astype(F32)
    if sigma <= 0:
        return m
    radius = int(4.0 * float(sigma) + 0.5)
    w = gaussian_kernel1d(float(sigma), radius)
    g = _correlate1d_nearest(m, w, axis=m.ndim - 2)
    g = _correlate1d_nearest(g, w, axis=m.ndim - 1)
    return np.maximum(m, g)


# ----------------------------------------------------------------------------------
# A4  token mask
# ----------------------------------------------------------------------------------
def token_mask(m1: np.ndarray, patch: int) -> np.ndarray:
    """valid[t] = any pixel of patch t lies outside m1 (a token is invalid
    iff all patch*patch pixels are masked).  Row-major over the token grid, the order
    of `flatten(2).transpose(1, 2)` at dstt.py:254.  (B, H, W) -> (B, T) bool."""
    m = np.asarray(m1).astype(bool)
    b, h, w = m.shape
    blocks = m.reshape(b, h // patch, patch, w // patch, patch)
    return (~blocks.all(axis=(2, 4))).reshape(b, -1)


# ----------------------------------------------------------------------------------
# A5  input conversion + redaction + concat
# ----------------------------------------------------------------------------------
def u8_to_unit(rgb_u8: np.ndarray) -> np.ndarray:
    """dstt.py:314-315: float(u8) / 255.0 as an IEEE fp32 divide, HWC -> CHW.
    (H, W, 3) or (B, H, W, 3) u8 -> (B, 3, H, W) f32."""
    a = np.asarray(rgb_u8)
    if a.ndim == 3:
        a = a[None]
    return (a.astype(F32) / F32(255.0)).transpose(0, 3, 1, 2).copy()


def pack_input(rgb01: np.ndarray, m1: np.ndarray) -> np.ndarray:
    """Network input (dstt.py:253): cat[rgb zeroed inside m1 (masks.py:145-154), m1]."""
    m = np.asarray(m1).astype(F32)[:, None]
    rgb = np.where(m > 0, F32(0.0), rgb01.astype(F32))
    return np.concatenate([rgb, m], axis=1)


# ----------------------------------------------------------------------------------
# A6-A13  the DSTT forward (dstt.py:224-268), fp32
# ----------------------------------------------------------------------------------
def state_dict_names(cfg):
    """`DsttModel.state_dict()` key order (dstt.py:231-244, :139-144, :102-109, :123-129)."""
    names = ["embed.weight", "embed.bias"]
    for i in range(len(cfg.blocks)):
        b = f"blocks.{i}."
        names += [b + "norm1.weight", b + "norm1.bias"]
        for proj in ("q_proj", "k_proj", "v_proj", "out_proj"):
            names += [b + f"attn.{proj}.weight", b + f"attn.{proj}.bias"]
        names += [b + "norm2.weight", b + "norm2.bias", b + "ffn.net.0.weight",
                  b + "ffn.net.0.bias", b + "ffn.net.2.weight", b + "ffn.net.2.bias"]
    return names + ["vec2patch.deconv.weight", "vec2patch.deconv.bias", "decode.0.weight",
                    "decode.0.bias", "decode.2.weight", "decode.2.bias"]


class Params:
    """Named view of the 72 positional DRWT tensors (state_dict order)."""

    def __init__(self, cfg, arrays):
        names = state_dict_names(cfg)
        assert len(names) == len(arrays)
        self.d = {n: np.asarray(a, F32) for n, a in zip(names, arrays)}

    def __getitem__(self, k):
        return self.d[k]


def layer_norm(x, w, b, eps=1e-5):
    """nn.LayerNorm (dstt.py:141,143): biased variance, eps 1e-5."""
    mu = x.mean(-1, keepdims=True, dtype=np.float64).astype(x.dtype)
    d = x - mu
    var = (d * d).mean(-1, keepdims=True, dtype=np.float64).astype(x.dtype)
    return d / np.sqrt(var + x.dtype.type(eps)) * w + b


def linear(x, w, b):
    return x @ w.T + b


def gelu(x):
    """nn.GELU() default approximate='none' (dstt.py:128): 0.5 x (1 + erf(x/sqrt 2))."""
    return (0.5 * x * (1.0 + _erf(x.astype(np.float64) / math.sqrt(2.0)))).astype(x.dtype)


def attention(q, k, v, key_bias=None):
    """scaled_dot_product (dstt.py:89-99): softmax(q k^T / sqrt(dh)) v.
    q (..., Tq, dh), k/v (..., Tk, dh); key_bias broadcastable to (..., Tq, Tk)."""
    tq = q.shape[-2]
    step = 1024                        # query chunks: bounded memory at 1024^2
    if tq > step:
        return np.concatenate([attention(q[..., i:i + step, :], k, v, key_bias)
                               for i in range(0, tq, step)], axis=-2)
    s = (q @ np.swapaxes(k, -1, -2)) * q.dtype.type(1.0 / math.sqrt(q.shape[-1]))
    if key_bias is not None:
        s = s + key_bias
    s = s - s.max(-1, keepdims=True)
    e = np.exp(s)
    return (e / e.sum(-1, keepdims=True)) @ v


def mha(p, pre, q_tok, kv_tok, heads, key_bias=None):
    """MultiHeadAttention.forward (dstt.py:111-120)."""
    b, tq, c = q_tok.shape
    tk = kv_tok.shape[1]
    dh = c // heads
    q = linear(q_tok, p[pre + "q_proj.weight"], p[pre + "q_proj.bias"])
    k = linear(kv_tok, p[pre + "k_proj.weight"], p[pre + "k_proj.bias"])
    v = linear(kv_tok, p[pre + "v_proj.weight"], p[pre + "v_proj.bias"])
    q = q.reshape(b, tq, heads, dh).transpose(0, 2, 1, 3)
    k = k.reshape(b, tk, heads, dh).transpose(0, 2, 1, 3)
    v = v.reshape(b, tk, heads, dh).transpose(0, 2, 1, 3)
    att = attention(q, k, v, key_bias).transpose(0, 2, 1, 3).reshape(b, tq, c)
    return linear(att, p[pre + "out_proj.weight"], p[pre + "out_proj.bias"])


def ffn(p, pre, x):
    """_FeedForward (dstt.py:123-133)."""
    h = gelu(linear(x, p[pre + "ffn.net.0.weight"], p[pre + "ffn.net.0.bias"]))
    return linear(h, p[pre + "ffn.net.2.weight"], p[pre + "ffn.net.2.bias"])


def _neg_inf_bias(valid):
    return np.where(valid, F32(0.0), F32(-np.inf)).astype(F32)


def spatial_block(p, pre, tokens, heads, valid=None):
    """SpatialBlock.forward (dstt.py:146-150).  Mask-aware (NEW): keys of
    invalid tokens get -inf unless the frame has no valid token (then unmasked);
    MAT update: every token becomes valid if any key was valid."""
    y = layer_norm(tokens, p[pre + "norm1.weight"], p[pre + "norm1.bias"])
    bias = None
    if valid is not None:
        anyv = valid.any(axis=1)
        eff = np.where(anyv[:, None], valid, True)
        bias = _neg_inf_bias(eff)[:, None, None, :]
        valid = valid | anyv[:, None]
    tokens = tokens + mha(p, pre + "attn.", y, y, heads, bias)
    tokens = tokens + ffn(p, pre, layer_norm(tokens, p[pre + "norm2.weight"],
                                             p[pre + "norm2.bias"]))
    return tokens, valid


def temporal_block(p, pre, tokens, slots, heads, groups, rows, cols, valid=None):
    """TemporalBlock.forward (dstt.py:177-195): LN1 of tokens and of both slots, split
    into `groups` contiguous row bands (`_band` :166-171), attend band queries to
    cat[band(cur), band(slot0), band(slot1)], unband (:173-175).  Mask-aware: current
    keys of invalid tokens get -inf, memory keys always valid; MAT update -> all valid."""
    b, t, c = tokens.shape
    for s in slots:
        if tuple(s.shape[-2:]) != (t, c):
            raise ValueError(f"memory slot shape {tuple(s.shape)} does not match tokens")
    n1w, n1b = p[pre + "norm1.weight"], p[pre + "norm1.bias"]
    tg = (rows // groups) * cols

    def band(x):
        return x.reshape(b * groups, tg, c)

    y = layer_norm(tokens, n1w, n1b)
    q = band(y)
    parts = [q]
    for s in slots:
        sb = s if s.ndim == 3 else np.broadcast_to(s[None], (b, t, c))
        parts.append(band(layer_norm(sb.astype(F32), n1w, n1b)))
    kv = np.concatenate(parts, axis=1)
    bias = None
    if valid is not None:
        kval = np.concatenate([valid.reshape(b * groups, tg),
                               np.ones((b * groups, 2 * tg), bool)], axis=1)
        bias = _neg_inf_bias(kval)[:, None, None, :]
        valid = np.ones_like(valid)
    att = mha(p, pre + "attn.", q, kv, heads, bias).reshape(b, t, c)
    tokens = tokens + att
    tokens = tokens + ffn(p, pre, layer_norm(tokens, p[pre + "norm2.weight"],
                                             p[pre + "norm2.bias"]))
    return tokens, valid


def patch_embed(p, x, patch):
    """DsttModel.patch_embed (dstt.py:246-254): Conv2d(4, C, k=p, s=p) as a per-patch
    GEMM; im2col order (c, ky, kx) = the conv weight's flatten order."""
    b, ci, h, w = x.shape
    r, cc = h // patch, w // patch
    cols = x.reshape(b, ci, r, patch, cc, patch).transpose(0, 2, 4, 1, 3, 5) \
            .reshape(b, r * cc, ci * patch * patch)
    wt = p["embed.weight"].reshape(p["embed.weight"].shape[0], -1)
    return cols @ wt.T + p["embed.bias"]


def vec2patch(p, tokens, rows, cols, patch, kernel, height, width):
    """Vec2Patch.forward (dstt.py:213-221): ConvTranspose2d(C, C, k, stride=patch) over
    the token grid (overlap-sum), crop offset (k - p)//2.  Restated as per-token patch
    GEMM + strided scatter-add, the same math as `tests/oracles.py:33-59` fold_oracle."""
    wt = p["vec2patch.deconv.weight"]                 # (C_in, C_out, k, k)
    ci, co = wt.shape[0], wt.shape[1]
    b = tokens.shape[0]
    pt = (tokens.reshape(b * rows * cols, ci) @ wt.reshape(ci, co * kernel * kernel)) \
        .reshape(b, rows, cols, co, kernel, kernel)
    fh, fw = (rows - 1) * patch + kernel, (cols - 1) * patch + kernel
    full = np.zeros((b, co, fh, fw), F32)
    for a in range(kernel):
        for c2 in range(kernel):
            full[:, :, a:a + rows * patch:patch, c2:c2 + cols * patch:patch] += \
                pt[:, :, :, :, a, c2].transpose(0, 3, 1, 2)
    full += p["vec2patch.deconv.bias"][None, :, None, None]
    o = (kernel - patch) // 2
    return full[:, :, o:o + height, o:o + width]


def conv3x3(x, w, bias):
    """nn.Conv2d(ci, co, 3, padding=1) (dstt.py:241,243): 9 shifted GEMMs, zero pad."""
    b, ci, h, wd = x.shape
    co = w.shape[0]
    xp = np.zeros((b, ci, h + 2, wd + 2), F32)
    xp[:, :, 1:-1, 1:-1] = x
    out = np.zeros((b, h, wd, co), F32)
    xt = xp.transpose(0, 2, 3, 1)
    for dy in range(3):
        for dx in range(3):
            out += xt[:, dy:dy + h, dx:dx + wd, :] @ w[:, :, dy, dx].T
    out += bias
    return out.transpose(0, 3, 1, 2)


def model_forward(cfg, params, rgb01, mask01, slots, token_valid=None):
    """DsttModel.forward (dstt.py:256-268) on the packed input.

    rgb01 (B,3,H,W) f32, mask01 (B,1,H,W) f32 -> (out01 (B,3,H,W), new_slot (B,T,C)).
    ``token_valid`` (B,T) bool switches on mask-aware attention."""
    p = params if isinstance(params, Params) else Params(cfg, params)
    if rgb01.shape[-2:] != (cfg.height, cfg.width):
        raise ValueError("input resolution does not match the model")
    x = np.concatenate([rgb01.astype(F32), mask01.astype(F32)], axis=1)
    tokens = patch_embed(p, x, cfg.patch).astype(F32)
    valid = None if token_valid is None else np.asarray(token_valid, bool).copy()
    for i, kind in enumerate(cfg.blocks):
        pre = f"blocks.{i}."
        if kind == "S":
            tokens, valid = spatial_block(p, pre, tokens, cfg.heads, valid)
        else:
            tokens, valid = temporal_block(p, pre, tokens, slots, cfg.heads,
                                           cfg.temporal_groups, cfg.token_rows,
                                           cfg.token_cols, valid)
    new_slot = tokens
    raster = vec2patch(p, tokens, cfg.token_rows, cfg.token_cols, cfg.patch, cfg.kernel,
                       cfg.height, cfg.width)
    h = conv3x3(raster, p["decode.0.weight"], p["decode.0.bias"])
    h = np.where(h >= 0, h, h * F32(0.2))             # LeakyReLU(0.2), dstt.py:242
    h = conv3x3(h, p["decode.2.weight"], p["decode.2.bias"])
    out = (np.tanh(h) + F32(1.0)) * F32(0.5)          # dstt.py:267
    return out.astype(F32), new_slot.astype(F32)


# ----------------------------------------------------------------------------------
# A16/A17  composite and output conversion
# ----------------------------------------------------------------------------------
def composite(fill01, frame01, alpha):
    """NEW fp32 alpha composite: out = a*fill + (1-a)*frame.
    With a binary alpha this is the reference's `out[m] = filled[m]` (base.py:87-88)."""
    a = alpha.astype(F32)[:, None]
    return (a * fill01.astype(F32) + (F32(1.0) - a) * frame01.astype(F32)).astype(F32)


def to_u8(out01):
    """dstt.py:324-325: mul(255).round() (half-to-even) .clamp(0,255) -> uint8,
    (B,3,H,W) -> (B,H,W,3)."""
    v = np.clip(np.rint(out01.astype(F32) * F32(255.0)), 0, 255).astype(np.uint8)
    return v.transpose(0, 2, 3, 1).copy()


def composite_u8(fill_u8, rgb_u8, alpha):
    """u8 composite for the reference API: alpha==0 keeps the input byte, alpha==1 takes
    the engine byte (exactly base.py:87-88 when alpha is binary), else
    rint(a*fill + (1-a)*rgb) in fp32."""
    a = alpha.astype(F32)[..., None]
    f = fill_u8.astype(F32)
    x = rgb_u8.astype(F32)
    mix = np.clip(np.rint(a * f + (F32(1.0) - a) * x), 0, 255).astype(np.uint8)
    return np.where(a == 0, rgb_u8, np.where(a == 1, fill_u8, mix))


# ----------------------------------------------------------------------------------
# the whole hot path
# ----------------------------------------------------------------------------------
def inpaint_path(cfg, params, rgb01, m0, slots):
    """mask -> dilate -> feather -> token mask -> forward -> composite (float API).

    rgb01 (B,3,H,W) f32 frame (raw or redacted), m0 (B,H,W) bool privacy mask,
    slots (slot0, slot1) each (T,C) or (B,T,C).  Returns a dict of every stage."""
    m0 = np.asarray(m0).astype(bool)
    m1 = dilate_mask(m0, cfg.mask_dilate)
    alpha = feather_mask(m1, cfg.mask_feather_sigma)
    tv = token_mask(m1, cfg.patch)
    x = pack_input(rgb01, m1)
    fill, new_slot = model_forward(cfg, params, x[:, :3], x[:, 3:],
                                   slots, tv if cfg.mask_aware_attention else None)
    out = composite(fill, rgb01, alpha)
    return {"m1": m1, "alpha": alpha, "token_valid": tv, "fill": fill,
            "slot": new_slot, "out": out}
