"""Generate golden fixtures from the REAL reference package (`dimreal`).

Run in the build container only (needs `/root/reference`, which never reaches the GPU
box):  python tests/golden/make_golden.py

Every fixture is the output of the unmodified reference on seeded inputs, or of the
reference's own primitives (scipy.ndimage with `masks._CROSS`) for the mask stages the
reference composes from them.  Mask-aware attention has no reference implementation;
its fixture comes from a shim around the reference model that adds -inf to invalid keys
inside `dstt.scaled_dot_product`.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REF))
sys.path.insert(0, str(REPO))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import torch  # noqa: E402
from scipy import ndimage  # noqa: E402

from dimreal import masks as ref_masks  # noqa: E402
from dimreal.inpaint import dstt as ref_dstt  # noqa: E402
from dimreal.inpaint.dstt import DsttConfig, DsttEngine, Vec2Patch  # noqa: E402
from dimreal.masks import BinaryMask  # noqa: E402

from paper_2509_10466_b200 import synth  # noqa: E402  (input generator only)

torch.set_num_threads(os.cpu_count() or 1)


def perturb_1d(engine: DsttEngine, seed: int) -> None:
    """Make biases and LayerNorm affine non-trivial (seeded init zeroes them)."""
    rng = np.random.default_rng(seed)
    with torch.no_grad():
        for _, p in engine.model.named_parameters():
            if p.dim() == 1:
                p.add_(torch.from_numpy(rng.normal(0.0, 0.1, p.shape).astype(np.float32)))


def weight_digest(engine: DsttEngine) -> np.ndarray:
    """Per-tensor (sum, sum of squares, first value) in float64, state_dict order."""
    rows = []
    for t in engine.model.state_dict().values():
        a = t.detach().numpy().astype(np.float64).ravel()
        rows.append([a.sum(), (a * a).sum(), a[0]])
    return np.array(rows)


def cfg_dict(cfg: DsttConfig) -> np.ndarray:
    return np.array([cfg.width, cfg.height, cfg.patch, cfg.channels, cfg.kernel,
                     cfg.heads, cfg.temporal_groups])


def save(name: str, **arrays) -> None:
    path = HERE / name
    np.savez_compressed(path, **arrays)
    print(f"{name}: {path.stat().st_size / 1024:.0f} KiB")


def gen_masks() -> None:
    rng = np.random.default_rng(2024)
    m0 = np.zeros((6, 45, 61), bool)
    m0[0] = rng.random((45, 61)) > 0.97                  # sparse specks
    m0[1, 10:30, 5:40] = True                             # block
    m0[2] = rng.random((45, 61)) > 0.6                    # dense noise
    m0[3, 0:3, :] = True                                  # touches the border
    m0[3, :, 58:] = True
    m0[4, 22, 30] = True                                  # single pixel
    m0[5] = synth.ellipse(45, 61, 20, 30, 9, 14)
    out = {"m0": m0}
    for r in (0, 1, 3, 5):
        d = np.stack([ndimage.binary_dilation(m, structure=ref_masks._CROSS,
                                              iterations=r) if r else m for m in m0])
        out[f"dilate_r{r}"] = d
    for sigma in (1.5, 3.0):
        m1 = out["dilate_r3"].astype(np.float32)
        g = np.stack([ndimage.gaussian_filter(m, sigma=sigma, mode="nearest", truncate=4.0)
                      for m in m1])
        out[f"feather_r3_s{sigma}"] = np.maximum(m1, g)
    save("masks.npz", **out)


def gen_attention() -> None:
    torch.manual_seed(3)
    q = torch.randn(2, 4, 37, 16)
    k = torch.randn(2, 4, 53, 16)
    v = torch.randn(2, 4, 53, 16)
    o, w = ref_dstt.scaled_dot_product(q, k, v)
    save("attention.npz", q=q.numpy(), k=k.numpy(), v=v.numpy(), out=o.numpy(),
         rowsum=w.sum(-1).numpy())


def gen_vec2patch() -> None:
    cfg = DsttConfig(width=64, height=48, channels=16, temporal_groups=2)
    torch.manual_seed(4)
    v2p = Vec2Patch(cfg, cfg.channels)
    tokens = torch.randn(1, cfg.tokens, cfg.channels)
    with torch.no_grad():
        ras = v2p(tokens)
    save("vec2patch.npz", cfg=cfg_dict(cfg), tokens=tokens.numpy(),
         weight=v2p.deconv.weight.detach().numpy(), bias=v2p.deconv.bias.detach().numpy(),
         raster=ras.numpy())


def gen_forward_b64() -> None:
    """Baseline network (patch 8, C 64, k 10, heads 4, groups 4) at 64x64, B=2,
    perturbed 1-D params, cold (zero) and warm (random per-stream) memory."""
    cfg = DsttConfig(width=64, height=64, temporal_groups=4)
    eng = DsttEngine(cfg, seed=11)
    seeded_digest = weight_digest(eng)
    perturb_1d(eng, 11)
    rng = np.random.default_rng(5)
    rgb = rng.random((2, 3, 64, 64)).astype(np.float32)
    mask = np.zeros((2, 1, 64, 64), np.float32)
    mask[0, 0, 10:40, 20:50] = 1
    mask[1, 0] = rng.random((64, 64)) > 0.8
    rgb = rgb * (1 - mask)
    cold = tuple(torch.zeros(1, cfg.tokens, cfg.channels).expand(2, -1, -1).contiguous()
                 for _ in range(2))
    warm = tuple(torch.from_numpy(rng.normal(0, 1, (2, cfg.tokens, cfg.channels))
                                  .astype(np.float32)) for _ in range(2))
    with torch.no_grad():
        out_c, slot_c = eng.model(torch.from_numpy(rgb), torch.from_numpy(mask), cold)
        out_w, slot_w = eng.model(torch.from_numpy(rgb), torch.from_numpy(mask), warm)
    save("forward_b64.npz", cfg=cfg_dict(cfg), weight_seed=11, perturb_seed=11,
         seeded_digest=seeded_digest, digest=weight_digest(eng), rgb=rgb, mask=mask,
         warm0=warm[0].numpy(), warm1=warm[1].numpy(), out_cold=out_c.numpy(),
         slot_cold=slot_c.numpy(), out_warm=out_w.numpy(), slot_warm=slot_w.numpy())


def gen_small_sequence() -> None:
    """Reference engine.inpaint (u8 API) on the small preset, 4 frames, memory carried."""
    cfg = DsttConfig.small()
    eng = DsttEngine(cfg, seed=1)
    rng = np.random.default_rng(31)
    mem = eng.zero_memory()
    rgbs, bits_all, outs, slots = [], [], [], []
    for t in range(4):
        rgb = rng.integers(0, 256, size=(36, 64, 3), dtype=np.uint8)
        bits = rng.random((36, 64)) > float(rng.uniform(0.5, 0.95))
        if t == 2:
            bits[:] = False                               # empty-mask frame
        rgb[bits] = 0
        res = eng.inpaint(rgb, BinaryMask(bits), mem)
        mem = res.memory
        rgbs.append(rgb)
        bits_all.append(bits)
        outs.append(res.rgb)
        slots.append(mem.slots[-1].numpy())
    save("small_sequence.npz", cfg=cfg_dict(cfg), weight_seed=1,
         digest=weight_digest(eng), rgb=np.stack(rgbs), bits=np.stack(bits_all),
         out=np.stack(outs), slot=np.stack(slots))


def gen_c1() -> None:
    """C1 (BASELINE configs[0]): 256^2, seed 0, r=5, sigma=3, seeded weights seed 0,
    cold memory.  The reference model runs on (rgb zeroed in m1, m1); m1/alpha from the
    reference primitives."""
    cfg = DsttConfig(width=256, height=256, temporal_groups=4)
    eng = DsttEngine(cfg, seed=0)
    img, m0 = synth.c1_frame(0, 256)
    m1 = ndimage.binary_dilation(m0, structure=ref_masks._CROSS, iterations=5)
    g = ndimage.gaussian_filter(m1.astype(np.float32), sigma=3.0, mode="nearest",
                                truncate=4.0)
    alpha = np.maximum(m1.astype(np.float32), g)
    rgb = img[None] * (1 - m1[None, None])
    zero = torch.zeros(1, cfg.tokens, cfg.channels)
    with torch.no_grad():
        out, slot = eng.model(torch.from_numpy(rgb.astype(np.float32)),
                              torch.from_numpy(m1[None, None].astype(np.float32)),
                              (zero, zero))
    out = out.numpy()
    comp = alpha[None, None] * out + (1 - alpha[None, None]) * img[None]
    save("c1_256.npz", digest=weight_digest(eng),
         img_sha=np.frombuffer(hashlib.sha256(img.tobytes()).digest(), np.uint8),
         m0=np.packbits(m0), m1=np.packbits(m1), alpha=alpha.astype(np.float16),
         out_f16=out.astype(np.float16), out_sum=np.float64(out.astype(np.float64).sum()),
         comp_f16=comp.astype(np.float16), slot_f16=slot.numpy().astype(np.float16))


class _KeyBiasShim:
    """Replaces dstt.scaled_dot_product so a per-block key bias can be injected."""

    def __init__(self):
        self.bias = None
        self.orig = ref_dstt.scaled_dot_product

    def __call__(self, q, k, v):
        scale = 1.0 / np.sqrt(q.shape[-1])
        s = torch.matmul(q, k.transpose(-2, -1)) * scale
        if self.bias is not None:
            s = s + self.bias
        w = torch.softmax(s, dim=-1)
        return torch.matmul(w, v), w


def gen_mask_aware() -> None:
    """Mask-aware attention (NEW) on the reference model through the shim:
    block 0 (S) masks keys of fully-masked tokens; MAT update -> later blocks unmasked."""
    cfg = DsttConfig(width=64, height=64, temporal_groups=4)
    eng = DsttEngine(cfg, seed=12)
    perturb_1d(eng, 12)
    rng = np.random.default_rng(8)
    rgb = rng.random((2, 3, 64, 64)).astype(np.float32)
    m = np.zeros((2, 64, 64), bool)
    m[0, 8:40, 16:56] = True                      # many fully-masked tokens
    m[1] = True                                   # fully masked frame: fallback path
    valid = ~m.reshape(2, 8, 8, 8, 8).all(axis=(2, 4)).reshape(2, -1)
    rgb = (rgb * (1 - m[:, None])).astype(np.float32)
    warm = tuple(torch.from_numpy(rng.normal(0, 1, (2, cfg.tokens, cfg.channels))
                                  .astype(np.float32)) for _ in range(2))
    shim = _KeyBiasShim()
    ref_dstt.scaled_dot_product = shim
    try:
        model = eng.model
        with torch.no_grad():
            tokens = model.patch_embed(torch.from_numpy(rgb),
                                       torch.from_numpy(m[:, None].astype(np.float32)))
            v = torch.from_numpy(valid)
            tg = cfg.tokens // cfg.temporal_groups
            for block in model.blocks:
                if isinstance(block, ref_dstt.TemporalBlock):
                    kv = torch.cat([v.reshape(2 * cfg.temporal_groups, tg),
                                    torch.ones(2 * cfg.temporal_groups, 2 * tg, dtype=bool)],
                                   dim=1)
                    shim.bias = torch.where(kv, 0.0, float("-inf"))[:, None, None, :]
                    tokens = block(tokens, warm)
                    v = torch.ones_like(v)
                else:
                    anyv = v.any(dim=1, keepdim=True)
                    eff = torch.where(anyv, v, torch.ones_like(v))
                    shim.bias = torch.where(eff, 0.0, float("-inf"))[:, None, None, :]
                    tokens = block(tokens)
                    v = v | anyv
            slot = tokens
            out = (torch.tanh(model.decode(model.vec2patch(tokens))) + 1.0) * 0.5
    finally:
        ref_dstt.scaled_dot_product = shim.orig
    save("mask_aware_b64.npz", cfg=cfg_dict(cfg), weight_seed=12, perturb_seed=12,
         digest=weight_digest(eng), rgb=rgb, m=m, valid=valid, warm0=warm[0].numpy(),
         warm1=warm[1].numpy(), out=out.numpy(), slot=slot.numpy())


def gen_frame_ops() -> None:
    """Display path, mask producer and point-cloud transplant outputs of the reference
    itself (pipeline.upscale2x / _composite_upscaled / transplant_pointcloud with their
    numba kernels, masks.merge_private_masks / redact)."""
    from dimreal import pipeline as ref_pipe
    from dimreal.detection import Detection2D, PrivacyState, TrackedObject
    from dimreal.scene import CameraIntrinsics
    from dimreal.scene import FrameRGBD

    rng = np.random.default_rng(2509)
    out = {}
    # upscale2x: ragged sizes, 1 and 3 channels
    for i, (h, w, c) in enumerate([(1, 1, 3), (3, 5, 3), (7, 9, 1), (36, 64, 3), (45, 130, 3)]):
        a = rng.integers(0, 256, size=(h, w, c) if c == 3 else (h, w), dtype=np.uint8)
        out[f"up_in{i}"] = a
        out[f"up_out{i}"] = ref_pipe.upscale2x(a)
    # display composite at a display-like size (ellipse blobs + stroke near the border)
    h, w = 90, 160
    original = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    inpainted = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    yy, xx = np.mgrid[0:h, 0:w]
    bits = ((yy - 40) ** 2 / 400 + (xx - 60) ** 2 / 900 < 1) | ((yy < 6) & (xx > 120))
    bits[:, 0] |= (yy[:, 0] > 70)
    mask = BinaryMask(bits)
    up_orig = ref_pipe.upscale2x(original)
    out.update(disp_original=original, disp_inpainted=inpainted, disp_mask=bits,
               disp_out=ref_pipe._composite_upscaled(up_orig, inpainted, mask))
    failed = up_orig.copy()
    failed[mask.upscale_nearest(2).bits] = 0
    out["disp_failed"] = failed
    # merge_private_masks + redact
    masks = rng.random((4, 24, 32)) > 0.7
    states = [PrivacyState.PRIVATE, PrivacyState.PUBLIC, PrivacyState.PRIVATE,
              PrivacyState.PUBLIC]
    tracks = [TrackedObject(id=i, class_label="thing",
                            latest=Detection2D.from_mask("thing", BinaryMask(m)), state=s)
              for i, (m, s) in enumerate(zip(masks, states))]
    merged = ref_masks.merge_private_masks(tracks, 32, 24)
    rgb = rng.integers(0, 256, size=(24, 32, 3), dtype=np.uint8)
    frame = FrameRGBD(rgb=rgb, depth=np.ones((24, 32), np.float32), frame_id=0, timestamp_ns=0)
    out.update(mr_masks=masks, mr_private=np.array([s is PrivacyState.PRIVATE for s in states]),
               mr_rgb=rgb, mr_merged=merged.bits, mr_redacted=ref_masks.redact(frame, merged).rgb)
    # point clouds: random valid set, all-invalid, single principal-point pixel
    intr = CameraIntrinsics(fx=100.0, fy=100.0, cx=32.0, cy=18.0, width=64, height=36)
    out["pc_intr"] = np.array([intr.fx, intr.fy, intr.cx, intr.cy])
    for i in range(3):
        depth = (rng.random((36, 64)) * 4).astype(np.float32)
        if i == 0:
            depth[depth < 1.5] = 0.0
        elif i == 1:
            depth[:] = 0.0
        else:
            depth[:] = 0.0
            depth[18, 32] = 2.0
        rgbp = rng.integers(0, 256, size=(36, 64, 3), dtype=np.uint8)
        cloud = ref_pipe.transplant_pointcloud(rgbp, depth, intr, frame_id=i)
        out.update({f"pc_depth{i}": depth, f"pc_rgb{i}": rgbp, f"pc_xyz{i}": cloud.xyz,
                    f"pc_col{i}": cloud.rgb})
    # a larger case with a non-integer principal point
    intr2 = CameraIntrinsics(fx=305.7, fy=304.9, cx=159.6, cy=90.3, width=320, height=180)
    depth = (rng.random((180, 320)) * 5).astype(np.float32)
    depth[rng.random((180, 320)) < 0.3] = 0.0
    rgbp = rng.integers(0, 256, size=(180, 320, 3), dtype=np.uint8)
    cloud = ref_pipe.transplant_pointcloud(rgbp, depth, intr2)
    out.update(pc_intr3=np.array([intr2.fx, intr2.fy, intr2.cx, intr2.cy]), pc_depth3=depth,
               pc_rgb3=rgbp, pc_xyz3=cloud.xyz, pc_col3=cloud.rgb)
    save("frame_ops.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:                       # regenerate only the named fixtures
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        sys.exit(0)
    gen_frame_ops()
    gen_masks()
    gen_attention()
    gen_vec2patch()
    gen_forward_b64()
    gen_small_sequence()
    gen_c1()
    gen_mask_aware()
