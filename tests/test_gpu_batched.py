"""GPU parity of the batch-throughput path (BASELINE configs[2] C3 and configs[4] C5).

At B*T >= ~18.9k tokens the token chains switch from the 32/64-token latency kernel
(`token_q_kernel`) to the 128-token throughput kernel (`token_tc_kernel`), and the last
block fills the new memory slot's K/V cache itself (engine.cu, `fill_here`) instead of
leaving it to the next forward's slot K/V launches.  These tests drive that code at the
real C3 / C5 shapes and, through the DR_TOK_ROWS override, on the reference goldens,
all against the CPU oracle: masks bit-exact, frames within max-abs 2e-2 and PSNR >= 40 dB
(BASELINE.json north_star).

Reference semantics: TemporalBlock with per-stream (B,T,C) slots `dstt.py:177-195`
(`:189` expand), SpatialBlock `:136-150`, DsttModel.forward `:256-268`.
"""

import numpy as np
import pytest

from conftest import cfg_from, golden, perturb_1d

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import dstt_oracle as O  # noqa: E402
from paper_2509_10466_b200 import DsttConfig, DsttEngine, synth  # noqa: E402
from paper_2509_10466_b200.weights import seed_parameters  # noqa: E402

MAX_ABS = 2e-2
MIN_PSNR = 40.0


def psnr(a, b):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10 * np.log10(1.0 / mse)


def check_img(got, ref, what):
    err = float(np.max(np.abs(got - ref)))
    p = psnr(got, ref)
    assert err <= MAX_ABS, f"{what}: max-abs {err:.3e}"
    assert p >= MIN_PSNR, f"{what}: PSNR {p:.1f} dB"
    return err


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def test_c5_batch8_512_cold_vs_oracle():
    """C5 shape: 8 independent 512^2 frames (32768 tokens -> 128-token tiles), cold
    memory, seeded C5 masks (rectangles / strokes / ellipse unions, 5-45 %)."""
    cfg = DsttConfig.baseline(512, mask_dilate=5, mask_feather_sigma=3.0)
    eng = DsttEngine(cfg, seed=0)
    B = 8
    assert eng.token_tile_rows(B) == 128, "C5 must run the 128-token throughput kernel"
    imgs, masks = synth.frame_pool("C5", B)
    res = eng.run(cuda(imgs), cuda(masks), None, want_fill=True, want_masks=True)
    w = O.Params(cfg, seed_parameters(cfg, 0))
    zero = np.zeros((cfg.tokens, cfg.channels), np.float32)
    out = res["out"].cpu().numpy()
    slot = res["slot"].cpu().numpy()
    m1 = res["m1"].cpu().numpy().astype(bool)
    tv = res["token_valid"].cpu().numpy().astype(bool)
    for i in range(B):
        ref = O.inpaint_path(cfg, w, imgs[i:i + 1], masks[i:i + 1], (zero, zero))
        assert np.array_equal(m1[i], ref["m1"][0]), f"frame {i} dilation"
        assert np.array_equal(tv[i], ref["token_valid"][0]), f"frame {i} token mask"
        check_img(out[i:i + 1], ref["out"], f"C5 frame {i}")
        assert np.max(np.abs(slot[i] - ref["slot"][0])) < 5e-2


def test_c3_eight_streams_batched_warm_memory_vs_oracle():
    """C3 shape: 8 video streams batched on one GPU with per-stream (B,T,C) memory, 3
    frames each.  Frame 2 reads slot K/V the engine computed inside frame 1's last block
    (cache hit, no slot K/V launch for it); frame 3 reads two such slots."""
    cfg = DsttConfig.baseline(512, mask_dilate=5, mask_feather_sigma=3.0)
    eng = DsttEngine(cfg, seed=0)
    S, F = 8, 3
    assert eng.token_tile_rows(S) == 128
    streams = [synth.C3Stream(s) for s in range(S)]
    w = O.Params(cfg, seed_parameters(cfg, 0))
    T, C = cfg.tokens, cfg.channels
    from paper_2509_10466_b200.memory import InpaintMemory
    mem = InpaintMemory.from_zero_slot(torch.zeros((S, T, C), device="cuda"))
    ref_slots = [(np.zeros((T, C), np.float32),) * 2 for _ in range(S)]
    launches = []
    for t in range(F):
        frames = [st.frame(t) for st in streams]
        img = np.stack([f[0] for f in frames])
        m0 = np.stack([f[1] for f in frames])
        res = eng.run(cuda(img), cuda(m0), mem.slots)
        launches.append(eng.kernels_per_forward())
        mem = mem.push(res["slot"])
        out = res["out"].cpu().numpy()
        for s in range(S):
            ref = O.inpaint_path(cfg, w, img[s:s + 1], m0[s:s + 1], ref_slots[s])
            ref_slots[s] = (ref_slots[s][1], ref["slot"][0])
            check_img(out[s:s + 1], ref["out"], f"C3 stream {s} frame {t}")
    # 1 mask + slot K/V (2 temporal blocks per uncached slot) + embed + 8 block kernels +
    # 3 decoder (fused tile pass, image border, seams): frames 0 and 1 project the (shared)
    # zero slot, frame 2 nothing (both slots were filled inside the previous forwards' last
    # blocks)
    base = 1 + 1 + 8 + 3
    assert launches == [base + 2, base + 2, base], launches


@pytest.mark.parametrize("rows", [128, 64, 32])
def test_forced_tile_rows_on_reference_golden(monkeypatch, rows):
    """Every token-kernel tile size, forced on the reference forward golden (B=2 at 64^2,
    perturbed biases / LayerNorm, cold and warm memory)."""
    monkeypatch.setenv("DR_TOK_ROWS", str(rows))        # read at engine creation
    g = golden("forward_b64.npz")
    cfg = cfg_from(g["cfg"])
    w = perturb_1d(seed_parameters(cfg, int(g["weight_seed"])), int(g["perturb_seed"]))
    eng = DsttEngine.from_arrays(cfg, w)
    assert eng.token_tile_rows(2) == rows
    zero = torch.zeros(cfg.tokens, cfg.channels)
    fill, slot = eng.model_forward(cuda(g["rgb"]), cuda(g["mask"]), (zero, zero))
    check_img(fill.cpu().numpy(), g["out_cold"], f"{rows}-row cold")
    assert np.max(np.abs(slot.cpu().numpy() - g["slot_cold"])) < 5e-2
    fill, slot = eng.model_forward(cuda(g["rgb"]), cuda(g["mask"]),
                                   (cuda(g["warm0"]), cuda(g["warm1"])))
    check_img(fill.cpu().numpy(), g["out_warm"], f"{rows}-row warm")
    assert np.max(np.abs(slot.cpu().numpy() - g["slot_warm"])) < 5e-2


def test_forced_128_rows_carried_memory_matches_oracle_and_small_tiles(monkeypatch):
    """Batch-1 frames through the 128-row kernel with engine-carried memory: the slot K/V
    the last block fills must equal a fresh projection (clone -> recompute) bit for bit,
    and the frames must match the oracle and the latency kernel's result."""
    cfg = DsttConfig.baseline(128, mask_dilate=2, mask_feather_sigma=1.5)
    imgs, masks = synth.frame_pool("C1", 4, size=128)
    w = seed_parameters(cfg, 5)
    monkeypatch.setenv("DR_TOK_ROWS", "128")
    big = DsttEngine.from_arrays(cfg, w)
    monkeypatch.delenv("DR_TOK_ROWS")
    small = DsttEngine.from_arrays(cfg, w)
    assert big.token_tile_rows(1) == 128 and small.token_tile_rows(1) < 128
    zero = np.zeros((cfg.tokens, cfg.channels), np.float32)
    ref_slots = (zero, zero)
    mem_b, mem_s = big.zero_memory(), small.zero_memory()
    for t in range(4):
        x, m = cuda(imgs[t:t + 1]), cuda(masks[t:t + 1])
        rb = big.run(x, m, mem_b.slots)
        rc = big.run(x, m, [s if big._is_zero_slot(s) else s.clone()     # no cache reuse
                            for s in mem_b.slots])
        assert torch.equal(rb["out"], rc["out"]) and torch.equal(rb["slot"], rc["slot"])
        rs = small.run(x, m, mem_s.slots)
        mem_b, mem_s = mem_b.push(rb["slot"][0]), mem_s.push(rs["slot"][0])
        ref = O.inpaint_path(cfg, O.Params(cfg, w), imgs[t:t + 1], masks[t:t + 1], ref_slots)
        ref_slots = (ref_slots[1], ref["slot"][0])
        check_img(rb["out"].cpu().numpy(), ref["out"], f"128-row frame {t}")
        check_img(rb["out"].cpu().numpy(), rs["out"].cpu().numpy(), f"128 vs small {t}")


@pytest.mark.parametrize("fused", ["1", "0"])
def test_both_decoders_on_reference_golden_and_small_frames(monkeypatch, fused):
    """The fused decoder (tile pass + border + seams) and the unfused sequence (Vec2Patch,
    decode.0 with decode.2's taps, gather) are both product paths (chosen by batch size,
    DR_DEC_FUSED forces one): each against the reference forward golden (64^2, B=2, all
    four image borders inside one tile) and the oracle at 128^2 (seams)."""
    monkeypatch.setenv("DR_DEC_FUSED", fused)
    g = golden("forward_b64.npz")
    cfg = cfg_from(g["cfg"])
    w = perturb_1d(seed_parameters(cfg, int(g["weight_seed"])), int(g["perturb_seed"]))
    eng = DsttEngine.from_arrays(cfg, w)
    fill, _ = eng.model_forward(cuda(g["rgb"]), cuda(g["mask"]),
                                (cuda(g["warm0"]), cuda(g["warm1"])))
    check_img(fill.cpu().numpy(), g["out_warm"], f"decoder {fused} golden")
    cfg = DsttConfig.baseline(128, mask_dilate=3, mask_feather_sigma=2.0)
    eng = DsttEngine(cfg, seed=0)
    imgs, masks = synth.frame_pool("C1", 2, size=128)
    res = eng.run(cuda(imgs), cuda(masks), None, want_fill=True)
    zero = np.zeros((cfg.tokens, cfg.channels), np.float32)
    ref = O.inpaint_path(cfg, seed_parameters(cfg, 0), imgs, masks, (zero, zero))
    check_img(res["fill"].cpu().numpy(), ref["fill"], f"decoder {fused} 128^2 fill")
    check_img(res["out"].cpu().numpy(), ref["out"], f"decoder {fused} 128^2 composite")


@pytest.mark.parametrize("fused", ["1", "0"])
def test_decoders_on_partial_tiles_256x136(monkeypatch, fused):
    """A non-square frame whose width is not a multiple of the fused decoder's 64-pixel
    tile: 256 x 136 (tiles of 128 x 64 px -> a last column of 8-pixel tiles; token grid
    32 x 17, bands of 136 tokens), batch 3 cold and then warm with per-frame memory, both
    decoders against the oracle (u8 path: masks bit-exact, frames within the gate)."""
    monkeypatch.setenv("DR_DEC_FUSED", fused)
    cfg = DsttConfig(width=136, height=256, temporal_groups=4, mask_dilate=3,
                     mask_feather_sigma=2.0)
    eng = DsttEngine(cfg, seed=1)
    rng = np.random.default_rng(11)
    imgs = rng.random((3, 3, 256, 136)).astype(np.float32)
    masks = np.zeros((3, 256, 136), bool)
    masks[0, 0:40, 100:136] = True                        # touches the right / top border
    masks[1, 120:140, 60:70] = True                       # straddles the tile seams
    masks[2, 200:256, 0:30] = True                        # bottom-left corner
    w = seed_parameters(cfg, 1)
    zero = np.zeros((cfg.tokens, cfg.channels), np.float32)
    res = eng.run(cuda(imgs), cuda(masks), None, want_masks=True)
    out = res["out"].cpu().numpy()
    slots = res["slot"]
    for i in range(3):
        ref = O.inpaint_path(cfg, w, imgs[i:i + 1], masks[i:i + 1], (zero, zero))
        assert np.array_equal(res["m1"][i].cpu().numpy().astype(bool), ref["m1"][0])
        check_img(out[i:i + 1], ref["out"], f"decoder {fused} 256x136 cold frame {i}")
    warm = torch.from_numpy(rng.normal(0, 1, (3, cfg.tokens, 64)).astype(np.float32)).cuda()
    res2 = eng.run(cuda(imgs), cuda(masks), (warm, slots))
    for i in range(3):
        ref = O.inpaint_path(cfg, w, imgs[i:i + 1], masks[i:i + 1],
                             (warm[i].cpu().numpy(), slots[i].cpu().numpy()))
        check_img(res2["out"][i:i + 1].cpu().numpy(), ref["out"], f"decoder {fused} 256x136 warm {i}")
