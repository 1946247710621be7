"""Pin the CPU oracle (`oracle/dstt_oracle.py`) to outputs of the real reference.

The fixtures in tests/golden/ were produced by tests/golden/make_golden.py from the
unmodified reference package (and scipy.ndimage with the reference's `_CROSS` element
for the mask primitives).  These tests run on CPU and never touch /root/reference.
"""

import numpy as np
import pytest

from conftest import cfg_from, digest, golden, perturb_1d
from oracle import dstt_oracle as O
from paper_2509_10466_b200 import DsttConfig
from paper_2509_10466_b200.weights import seed_parameters


def test_seeded_weights_match_reference_digest():
    g = golden("forward_b64.npz")
    cfg = cfg_from(g["cfg"])
    w = seed_parameters(cfg, int(g["weight_seed"]))
    assert len(w) == 72
    np.testing.assert_allclose(digest(w), g["seeded_digest"], rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(digest(perturb_1d(w, int(g["perturb_seed"]))), g["digest"],
                               rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("r", [0, 1, 3, 5])
def test_dilate_bit_exact_vs_reference_cross(r):
    g = golden("masks.npz")
    assert np.array_equal(O.dilate_mask(g["m0"], r), g[f"dilate_r{r}"])


def test_dilation_growth_is_diamond():
    """tests/oracles.py:82-84 diamond_area: single pixel dilated k times."""
    for k in range(8):
        m = np.zeros((1, 41, 41), bool)
        m[0, 20, 20] = True
        assert O.dilate_mask(m, k).sum() == 2 * k * k + 2 * k + 1


@pytest.mark.parametrize("sigma", [1.5, 3.0])
def test_feather_vs_reference_scipy(sigma):
    g = golden("masks.npz")
    a = O.feather_mask(g["dilate_r3"], sigma)
    assert np.max(np.abs(a - g[f"feather_r3_s{sigma}"])) <= 1e-6
    assert (a[g["dilate_r3"]] == 1.0).all()


def test_token_mask_definition():
    m = np.zeros((1, 16, 24), bool)
    m[0, 0:8, 0:8] = True          # token 0 fully masked
    m[0, 8:16, 8:15] = True        # token 4 has one unmasked column
    v = O.token_mask(m, 8)
    assert v.shape == (1, 6)
    assert v.tolist() == [[False, True, True, True, True, True]]


def test_attention_vs_reference():
    g = golden("attention.npz")
    out = O.attention(g["q"], g["k"], g["v"])
    assert np.max(np.abs(out - g["out"])) < 1e-5


def test_vec2patch_vs_reference():
    g = golden("vec2patch.npz")
    cfg = cfg_from(g["cfg"])

    class P(dict):
        pass
    p = {"vec2patch.deconv.weight": g["weight"], "vec2patch.deconv.bias": g["bias"]}
    out = O.vec2patch(p, g["tokens"], cfg.token_rows, cfg.token_cols, cfg.patch,
                      cfg.kernel, cfg.height, cfg.width)
    assert np.max(np.abs(out - g["raster"])) < 1e-5


def _b64_params(g):
    cfg = cfg_from(g["cfg"])
    w = perturb_1d(seed_parameters(cfg, int(g["weight_seed"])), int(g["perturb_seed"]))
    return cfg, w


def test_forward_cold_and_warm_vs_reference():
    g = golden("forward_b64.npz")
    cfg, w = _b64_params(g)
    zero = np.zeros((cfg.tokens, cfg.channels), np.float32)
    out, slot = O.model_forward(cfg, w, g["rgb"], g["mask"], (zero, zero))
    assert np.max(np.abs(out - g["out_cold"])) < 1e-4
    assert np.max(np.abs(slot - g["slot_cold"])) < 1e-4
    out, slot = O.model_forward(cfg, w, g["rgb"], g["mask"], (g["warm0"], g["warm1"]))
    assert np.max(np.abs(out - g["out_warm"])) < 1e-4
    assert np.max(np.abs(slot - g["slot_warm"])) < 1e-4


def test_mask_aware_vs_reference_shim():
    g = golden("mask_aware_b64.npz")
    cfg, w = _b64_params(g)
    m = g["m"]
    assert np.array_equal(O.token_mask(m, 8), g["valid"])
    out, slot = O.model_forward(cfg, w, g["rgb"], m[:, None].astype(np.float32),
                                (g["warm0"], g["warm1"]), token_valid=g["valid"])
    assert np.max(np.abs(out - g["out"])) < 1e-4
    assert np.max(np.abs(slot - g["slot"])) < 1e-4


def test_small_preset_u8_sequence_vs_reference():
    """Reference engine.inpaint (u8 API, binary composite, memory FIFO) on 4 frames."""
    g = golden("small_sequence.npz")
    cfg = cfg_from(g["cfg"])
    w = seed_parameters(cfg, int(g["weight_seed"]))
    np.testing.assert_allclose(digest(w), g["digest"], rtol=1e-6, atol=1e-6)
    zero = np.zeros((cfg.tokens, cfg.channels), np.float32)
    slots = (zero, zero)
    for t in range(4):
        rgb, bits = g["rgb"][t], g["bits"][t]
        x = O.u8_to_unit(rgb)
        fill, slot = O.model_forward(cfg, w, x, bits[None, None].astype(np.float32), slots)
        out = O.composite_u8(O.to_u8(fill)[0], rgb, bits.astype(np.float32))
        # rounding to u8 can flip by one code where fp32 sums differ in the last ulp
        assert np.max(np.abs(out.astype(int) - g["out"][t].astype(int))) <= 1
        assert np.mean(out != g["out"][t]) < 1e-3
        assert np.max(np.abs(slot[0] - g["slot"][t])) < 1e-4
        slots = (slots[1], slot[0])


def test_c1_full_path_vs_reference():
    """BASELINE configs[0]: 256^2, r=5, sigma=3, seeded weights, cold memory."""
    from paper_2509_10466_b200 import synth
    import hashlib
    g = golden("c1_256.npz")
    cfg = DsttConfig.baseline(256, mask_dilate=5, mask_feather_sigma=3.0)
    w = seed_parameters(cfg, 0)
    np.testing.assert_allclose(digest(w), g["digest"], rtol=1e-6, atol=1e-6)
    img, m0 = synth.c1_frame(0, 256)
    assert hashlib.sha256(img.tobytes()).digest() == bytes(g["img_sha"])
    assert np.array_equal(np.packbits(m0), g["m0"])
    zero = np.zeros((cfg.tokens, cfg.channels), np.float32)
    res = O.inpaint_path(cfg, w, img[None], m0[None], (zero, zero))
    assert np.array_equal(np.packbits(res["m1"][0]), g["m1"])
    assert np.max(np.abs(res["alpha"][0] - g["alpha"].astype(np.float32))) < 1e-3
    assert np.max(np.abs(res["fill"] - g["out_f16"].astype(np.float32))) < 1e-3
    assert abs(float(res["fill"].astype(np.float64).sum()) - float(g["out_sum"])) < 1e-2
    assert np.max(np.abs(res["out"] - g["comp_f16"].astype(np.float32))) < 1e-3


# ------------------------------------------------------------------ frame byte kernels
def test_frame_ops_oracle_vs_reference_fixtures():
    """The numpy restatements of upscale2x / _composite_upscaled / merge+redact /
    pack_pointcloud reproduce the reference's own outputs bit for bit."""
    from oracle import frame_ops_oracle as F
    g = golden("frame_ops.npz")
    for i in range(5):
        assert np.array_equal(F.upscale2x(g[f"up_in{i}"]), g[f"up_out{i}"]), i
    assert np.array_equal(F.display_output(g["disp_original"], g["disp_inpainted"],
                                           g["disp_mask"]), g["disp_out"])
    assert np.array_equal(F.display_output(g["disp_original"], g["disp_inpainted"],
                                           g["disp_mask"], engine_failed=True), g["disp_failed"])
    merged = F.merge_private_masks(g["mr_masks"], g["mr_private"])
    assert np.array_equal(merged, g["mr_merged"])
    assert np.array_equal(F.redact(g["mr_rgb"], merged), g["mr_redacted"])
    for i in range(4):
        fx, fy, cx, cy = g["pc_intr3"] if i == 3 else g["pc_intr"]
        xyz, col = F.pack_pointcloud(g[f"pc_depth{i}"], g[f"pc_rgb{i}"], fx, fy, cx, cy)
        assert np.array_equal(xyz, g[f"pc_xyz{i}"]) and np.array_equal(col, g[f"pc_col{i}"]), i
