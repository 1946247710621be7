"""CUDA-IPC engine transport (paper_2509_10466_b200/service.py).

CPU: the protocol and memory semantics with a fake engine on shared CPU tensors (two
processes).  GPU: frames through a real engine process equal the in-process engine's
outputs bit for bit, memory carried per connection, errors mapped to the reference
exceptions."""

import numpy as np
import pytest

from paper_2509_10466_b200.errors import InputError, ProtocolError
from paper_2509_10466_b200.service import IpcEngineServer


class _FakeEngine:
    """out = rgb with the masked pixels set to the frame counter (memory = #pushes)."""
    height, width = 6, 8

    def zero_memory(self):
        from paper_2509_10466_b200.memory import InpaintMemory
        import torch
        return InpaintMemory.from_zero_slot(torch.zeros(2, 2))

    def run(self, rgb, mask, slots, out):
        import torch
        if (rgb[0][mask[0].bool()] != 0).any():
            raise InputError("input is not redacted: nonzero pixels inside mask")
        count = float(slots[1][0, 0]) + 1.0
        o = rgb[0].clone()
        o[mask[0].bool()] = int(count)
        out["out"][0].copy_(o)
        return {"out": out["out"], "slot": torch.full((1, 2, 2), count), "ms": 0.1}


def _fake_factory():
    return _FakeEngine()


def test_ipc_protocol_memory_and_errors_cpu():
    srv = IpcEngineServer(_fake_factory, device="cpu").start()
    cli = srv.connect()
    try:
        rng = np.random.default_rng(0)
        rgb = rng.integers(1, 256, (6, 8, 3), dtype=np.uint8)
        mask = np.zeros((6, 8), bool)
        mask[2:4, 3:6] = True
        rgb[mask] = 0
        outs = [cli.inpaint_frame(i, rgb, mask).rgb for i in range(3)]
        for i, o in enumerate(outs):                      # memory advances per request
            assert (o[mask] == i + 1).all() and np.array_equal(o[~mask], rgb[~mask])
        cli.reset()                                       # memory resets
        assert (cli.inpaint_frame(9, rgb, mask).rgb[mask] == 1).all()
        bad = rgb.copy()
        bad[2, 3] = 7
        with pytest.raises(InputError):
            cli.inpaint_frame(10, bad, mask)
        with pytest.raises(ProtocolError):
            cli.inpaint_frame(11, rgb[:4], mask[:4])
    finally:
        cli.close()
        srv.stop()


def _b200_factory():
    from paper_2509_10466_b200 import DsttConfig, DsttEngine
    return DsttEngine(DsttConfig.baseline(256, mask_dilate=5, mask_feather_sigma=3.0), seed=0)


@pytest.mark.gpu
def test_ipc_transport_matches_in_process_engine():
    from paper_2509_10466_b200 import synth
    from paper_2509_10466_b200.masks import BinaryMask
    ref = _b200_factory()
    srv = IpcEngineServer(_b200_factory).start()
    cli = srv.connect()
    try:
        mem = ref.zero_memory()
        for i in range(4):
            img, m = synth.c1_frame(i, 256)
            rgb = np.ascontiguousarray(np.clip(np.rint(img.transpose(1, 2, 0) * 255), 0, 255)
                                       .astype(np.uint8))
            rgb[m] = 0
            want = ref.inpaint(rgb, BinaryMask(m), mem)
            mem = want.memory
            got = cli.inpaint_frame(i, rgb, BinaryMask(m))
            assert np.array_equal(got.rgb, want.rgb), i
            assert got.inference_ms > 0
        rgb[m] = 255                                      # unredacted -> InputError
        with pytest.raises(InputError):
            cli.inpaint_frame(99, rgb, BinaryMask(m))
    finally:
        cli.close()
        srv.stop()
