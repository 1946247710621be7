"""GPU: BatchStreamer (overlapped upload / forward / download, streaming.py) equals the
serial DsttEngine.run on every batch, bit for bit, with and without carried per-stream
memory, and reports a batch's redaction error like run() does (base.py:76-79)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2509_10466_b200 import DsttConfig, DsttEngine, InputError  # noqa: E402
from paper_2509_10466_b200.streaming import BatchStreamer  # noqa: E402


def _batches(rng, n, B, H, W):
    out = []
    for _ in range(n):
        rgb = rng.integers(0, 256, size=(B, H, W, 3), dtype=np.uint8)
        m = np.zeros((B, H, W), np.uint8)
        for b in range(B):
            y, x = rng.integers(0, H // 2), rng.integers(0, W // 2)
            m[b, y:y + rng.integers(8, H // 2), x:x + rng.integers(8, W // 2)] = 1
        rgb[m.astype(bool)] = 0                                  # redacted input
        out.append((torch.from_numpy(rgb).pin_memory(), torch.from_numpy(m).pin_memory()))
    return out


@pytest.mark.parametrize("carried", [False, True])
def test_streamer_equals_serial_run(carried):
    cfg = DsttConfig.baseline(128, mask_dilate=3, mask_feather_sigma=1.5)
    B, n = 4, 5
    data = _batches(np.random.default_rng(7), n, B, 128, 128)
    eng, ref = DsttEngine(cfg, seed=0), DsttEngine(cfg, seed=0)
    bs = BatchStreamer(eng, B)
    outs = [torch.empty((B, 128, 128, 3), dtype=torch.uint8).pin_memory() for _ in range(n)]
    mem, rmem, slots, ref_res = None, None, [], []
    for k, (rgb, m) in enumerate(data):
        slot = bs.submit(rgb, m, outs[k], mem)
        r = ref.run(rgb, m, rmem)                                # serial, synchronous
        slots.append(slot)
        ref_res.append((r["out"].cpu(), r["slot"].cpu()))
        if carried:
            mem = (mem[1] if mem else torch.zeros_like(slot), slot)
            rmem = (rmem[1] if rmem else torch.zeros_like(r["slot"]), r["slot"])
    bs.finish()
    for k in range(n):
        assert torch.equal(outs[k], ref_res[k][0]), f"batch {k} composite"
        assert torch.equal(slots[k].cpu(), ref_res[k][1]), f"batch {k} new slot"


def test_streamer_reports_unredacted_batch():
    cfg = DsttConfig.baseline(64)
    B = 2
    data = _batches(np.random.default_rng(3), 3, B, 64, 64)
    rgb, m = data[1]
    rgb[1][m[1].bool()] = 200                                   # batch 1, frame 1 not redacted
    eng = DsttEngine(cfg, seed=0)
    bs = BatchStreamer(eng, B)
    out = torch.empty((B, 64, 64, 3), dtype=torch.uint8).pin_memory()
    with pytest.raises(InputError):
        for rgb_k, m_k in data:
            bs.submit(rgb_k, m_k, out)
        bs.finish()


@pytest.mark.parametrize("B", [1, 2])
def test_carried_streamer_graph_replays_equal_serial_run(B):
    """carry_memory=True: the streamer's own 2-slot FIFO per stream and, after the warm-up,
    CUDA-graph replays of the forward (one per buffer set x memory-ring phase, period 6)
    over two full periods -- bit-equal to the serial engine with the same FIFO."""
    cfg = DsttConfig.baseline(128, mask_dilate=3, mask_feather_sigma=1.5)
    n = BatchStreamer.GRAPH_WARM + 13
    data = _batches(np.random.default_rng(11), n, B, 128, 128)
    eng, ref = DsttEngine(cfg, seed=0), DsttEngine(cfg, seed=0)
    bs = BatchStreamer(eng, B, carry_memory=True)
    outs = [torch.empty((B, 128, 128, 3), dtype=torch.uint8).pin_memory() for _ in range(n)]
    zero = ref.zero_memory().slots[0]
    hist, ref_out, slots = [], [], []
    for k, (rgb, m) in enumerate(data):
        slot = bs.submit(rgb, m, outs[k])
        with torch.cuda.stream(bs.comp):                      # ring buffer: copy it in order
            slots.append(slot.clone())
        mem = (hist[-2] if k >= 2 else zero, hist[-1] if k >= 1 else zero)
        r = ref.run(rgb, m, mem)
        hist.append(r["slot"])
        ref_out.append(r["out"].cpu())
    bs.finish()
    torch.cuda.synchronize()
    assert len(bs.graphs) == 6
    for k in range(n):
        assert torch.equal(outs[k], ref_out[k]), f"frame {k} composite"
        assert torch.equal(slots[k].cpu(), hist[k].cpu()), f"frame {k} new slot"
