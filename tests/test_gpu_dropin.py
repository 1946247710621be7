"""The drop-in boundary driven by the REFERENCE's own caller.

`dimreal.service.LocalEngineClient` (service.py:191-210, the in-process client that
`Pipeline.step` calls at pipeline.py:297) from the unmodified reference installed in
`baseline/_ref` (baseline/install_ref.sh; it travels with the repo snapshot) drives this
repository's `DsttEngine` exactly as it drives the reference `DsttEngine`:
`engine.zero_memory()`, then `engine.inpaint(rgb, mask, memory)` -> EngineResult with
`.rgb`, `.memory`, `.inference_ms` (base.py:52-89).  The engine routes that call through
the C-ABI host call `dr_inpaint_u8_host_mem` (explicit memory slots).
"""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
if not (REF / "dimreal").is_dir():  # pragma: no cover
    pytest.skip("reference not installed (baseline/install_ref.sh)", allow_module_level=True)
sys.path.insert(0, str(REF))

from dimreal.masks import BinaryMask as RefBinaryMask  # noqa: E402
from dimreal.service import LocalEngineClient  # noqa: E402

from oracle import dstt_oracle as O  # noqa: E402
from paper_2509_10466_b200 import DsttConfig, DsttEngine, InputError, synth  # noqa: E402
from paper_2509_10466_b200.weights import seed_parameters  # noqa: E402


def _frames(n, size, seed=0):
    rng = np.random.default_rng(seed)
    imgs, masks = synth.frame_pool("C1", n, size=size)
    out = []
    for i in range(n):
        rgb = np.clip(np.rint(imgs[i].transpose(1, 2, 0) * 255), 0, 255).astype(np.uint8)
        bits = masks[i].copy()
        if i == 2:
            bits[:] = False                                  # empty mask frame
        if i == 3:
            bits |= rng.random(bits.shape) < 0.02            # ragged specks
        rgb[bits] = 0                                        # the pipeline redacts first
        out.append((rgb, bits))
    return out


def test_reference_local_engine_client_drives_the_engine():
    cfg = DsttConfig.baseline(128, mask_dilate=3, mask_feather_sigma=2.0)
    eng = DsttEngine(cfg, seed=0)
    client = LocalEngineClient(eng)                          # reference code
    frames = _frames(9, 128)
    w = O.Params(cfg, seed_parameters(cfg, 0))
    zero = np.zeros((cfg.tokens, cfg.channels), np.float32)
    ref_slots = (zero, zero)
    dev_mem = eng.zero_memory()
    for i, (rgb, bits) in enumerate(frames):
        call = client.inpaint_frame(i, rgb, RefBinaryMask(bits))   # reference BinaryMask
        assert call.rgb.shape == rgb.shape and call.rgb.dtype == np.uint8
        assert call.inference_ms > 0
        assert client.memory.pushes == i + 1
        # bit-equal to the batched device path with the same memory
        res = eng.run(torch.from_numpy(rgb)[None], torch.from_numpy(bits)[None],
                      dev_mem.slots)
        dev_mem = dev_mem.push(res["slot"][0])
        assert np.array_equal(call.rgb, res["out"][0].cpu().numpy()), f"frame {i}"
        assert torch.equal(client.memory.slots[1], res["slot"][0])
        # and within the north_star gate of the fp32 oracle composite
        rgb01 = O.u8_to_unit(rgb)
        ref = O.inpaint_path(cfg, w, rgb01, bits[None], ref_slots)
        ref_slots = (ref_slots[1], ref["slot"][0])
        got01 = call.rgb.transpose(2, 0, 1)[None] / 255.0
        assert np.max(np.abs(got01 - ref["out"])) <= 2e-2
        if not bits.any():
            assert np.array_equal(call.rgb, rgb)              # base.py:71-74
        keep = ref["alpha"][0] == 0
        assert np.array_equal(call.rgb[keep], rgb[keep])      # composite guarantee
    # the caller keeps only the latest memory: the engine recycles a few slot buffers
    assert len(eng._slot_pool) <= 4


def test_held_memories_are_never_overwritten():
    """Memory is an immutable value (memory.py:40-45): a memory the caller still holds
    keeps its slot contents while the engine goes on producing new slots."""
    cfg = DsttConfig.baseline(64)
    eng = DsttEngine(cfg, seed=1)
    frames = _frames(6, 64, seed=3)
    mem = eng.zero_memory()
    held = []
    for rgb, bits in frames:
        r = eng.inpaint(rgb, RefBinaryMask(bits), mem)
        held.append((r.memory, [s.clone() for s in r.memory.slots]))
        mem = r.memory
    for m, snap in held:
        for a, b in zip(m.slots, snap):
            assert torch.equal(a, b)
    view = mem.slots[1][:4]                                   # a view of a slot's storage
    snap = view.clone()
    mem_keep = mem
    del mem
    for rgb, bits in frames[:3]:
        mem_keep = eng.inpaint(rgb, RefBinaryMask(bits), mem_keep).memory
    assert torch.equal(view, snap)


def test_dropin_errors_propagate_through_the_reference_client():
    cfg = DsttConfig.baseline(64)
    eng = DsttEngine(cfg, seed=0)
    client = LocalEngineClient(eng)
    rgb = np.full((64, 64, 3), 9, np.uint8)
    bits = np.zeros((64, 64), bool)
    bits[5:20, 5:30] = True
    with pytest.raises(InputError):                          # not redacted (base.py:76-79)
        client.inpaint_frame(0, rgb, RefBinaryMask(bits))
    assert client.memory.pushes == 0                          # memory not advanced
    rgb[bits] = 0
    call = client.inpaint_frame(1, rgb, RefBinaryMask(bits))
    assert client.memory.pushes == 1 and call.rgb.shape == rgb.shape


def test_integration_md_ctypes_stub_runs_with_reference_classes():
    """INTEGRATION.md §B is executable: its ctypes binding, loaded as a module of the
    reference package (`dimreal.inpaint.b200`, relative imports of the reference's errors,
    base and memory), builds an engine from the reference DsttEngine's state_dict and is
    driven by the reference LocalEngineClient with real memory (NULL zero slot, pushed
    device slots).  Its frames equal this repository's DsttEngine.inpaint bit for bit."""
    import importlib.util
    import re

    from dimreal.inpaint import dstt as ref_dstt

    from paper_2509_10466_b200 import _lib
    text = (Path(__file__).resolve().parents[1] / "INTEGRATION.md").read_text()
    sec = text[text.index("## B. Bind the C-ABI directly"):text.index("## C.")]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    code = code.replace('ctypes.CDLL("libdrb200.so")', f'ctypes.CDLL("{_lib.LIB_PATH}")')
    spec = importlib.util.spec_from_loader("dimreal.inpaint.b200", loader=None)
    mod = importlib.util.module_from_spec(spec)
    mod.__package__ = "dimreal.inpaint"
    exec(compile(code, "INTEGRATION.md#B", "exec"), mod.__dict__)

    ref_cfg = ref_dstt.DsttConfig(width=64, height=64, temporal_groups=4)
    stub = mod.B200DsttEngine(ref_dstt.DsttEngine(ref_cfg, seed=0), mask_dilate=3,
                              feather_sigma=2.0)
    ours = DsttEngine(DsttConfig.baseline(64, mask_dilate=3, mask_feather_sigma=2.0), seed=0)
    client = LocalEngineClient(stub)
    mem = ours.zero_memory()
    for i, (rgb, bits) in enumerate(_frames(5, 64, seed=7)):
        call = client.inpaint_frame(i, rgb, RefBinaryMask(bits))
        r = ours.inpaint(rgb, RefBinaryMask(bits), mem)
        mem = r.memory
        assert np.array_equal(call.rgb, r.rgb), f"frame {i}"
        assert client.memory.pushes == i + 1
        assert torch.equal(client.memory.slots[1], r.memory.slots[1])
    rgb, bits = _frames(1, 64, seed=8)[0]
    rgb[bits] = 5
    if bits.any():
        with pytest.raises(Exception) as ei:
            stub.inpaint(rgb, RefBinaryMask(bits), stub.zero_memory())
        assert "redacted" in str(ei.value)
