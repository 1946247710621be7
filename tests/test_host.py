"""CPU tests of the host side: the reference-API types (config, memory FIFO, DRWT weights,
masks), the synthetic BASELINE generators, and the C-ABI library (loads, exports every
symbol include/dr_b200.h declares, struct layouts) -- no GPU compute.

Cases mirror the reference suite: test_dstt.py:15-38 (config), test_loss_weights.py:75-170
(memory FIFO, DRWT), test_masks.py:81-162 (redact, cross dilation/erosion growth)."""

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import REPO
from paper_2509_10466_b200 import (BinaryMask, ConfigError, DegenerateMaskError, DsttConfig,
                                   InpaintMemory, InputError, adjust_mask_area, load_weights,
                                   memory_push, redact, save_weights, synth)
from paper_2509_10466_b200 import _lib
from paper_2509_10466_b200.weights import check_shapes, parameter_specs, seed_parameters

HEADER = REPO / "include" / "dr_b200.h"


# ------------------------------------------------------------------ config
class TestConfig:
    def test_defaults_match_reference(self):
        c = DsttConfig()
        assert (c.width, c.height, c.patch, c.channels, c.kernel, c.heads,
                c.temporal_groups, c.blocks) == (640, 360, 8, 64, 10, 4, 3, ("S", "T", "S", "T"))
        assert (c.mask_dilate, c.mask_feather_sigma, c.mask_aware_attention) == (0, 0.0, False)

    def test_small_preset(self):
        s = DsttConfig.small()
        assert (s.width, s.height, s.tokens) == (64, 36, 144)

    @pytest.mark.parametrize("kw", [dict(width=65, height=36, patch=4),
                                    dict(width=64, height=64, heads=3),
                                    dict(width=64, height=64, kernel=4),
                                    dict(width=64, height=64, temporal_groups=3),
                                    dict(width=64, height=64, blocks=()),
                                    dict(width=64, height=64, blocks=("S", "X")),
                                    dict(width=64, height=64, mask_dilate=-1),
                                    dict(width=64, height=64, mask_feather_sigma=-1.0)])
    def test_invalid_rejected(self, kw):
        with pytest.raises(ConfigError):
            DsttConfig(**kw)

    def test_baseline_default_groups_invalid_at_512(self):
        """the reference default temporal_groups=3 is invalid at 512^2."""
        with pytest.raises(ConfigError):
            DsttConfig(width=512, height=512)
        assert DsttConfig.baseline(512).temporal_groups == 4

    def test_json_roundtrip(self):
        c = DsttConfig.baseline(256, mask_dilate=5, mask_feather_sigma=3.0,
                                mask_aware_attention=True)
        assert DsttConfig.from_dict(c.to_dict()) == c
        assert c.feather_radius == 12


# ------------------------------------------------------------------ memory FIFO
class TestMemory:
    def test_push_sequence_and_hundred_pushes(self):
        zero = np.zeros((2, 2), np.float32)
        mem = InpaintMemory.from_zero_slot(zero)
        sentinels = [np.full_like(zero, float(i)) for i in range(100)]
        for s in sentinels:
            mem = memory_push(mem, s)
        assert np.array_equal(mem.slots[0], sentinels[-2])
        assert np.array_equal(mem.slots[1], sentinels[-1])
        assert mem.pushes == 100 and mem.warm

    def test_slot_count_and_shape(self):
        with pytest.raises(ConfigError):
            InpaintMemory((np.zeros(3),))
        with pytest.raises(ConfigError):
            InpaintMemory((np.zeros(3), np.zeros(4)))
        mem = InpaintMemory.from_zero_slot(np.zeros((4, 4)))
        with pytest.raises(ConfigError):
            mem.push(np.zeros((4, 5)))


# ------------------------------------------------------------------ DRWT weights
class TestWeights:
    def test_roundtrip_bit_exact(self, rng, tmp_path):
        arrays = [rng.normal(size=s).astype(np.float32) for s in [(3, 4), (7,), (2, 3, 2, 2)]]
        save_weights(arrays, tmp_path / "w.drwt")
        for a, b in zip(arrays, load_weights(tmp_path / "w.drwt")):
            assert np.array_equal(a, b)

    @pytest.mark.parametrize("corrupt,match", [(lambda d: d.__setitem__(0, d[0] ^ 0xFF), "magic"),
                                               (lambda d: d.__setitem__(4, 9), "version")])
    def test_corruption(self, tmp_path, corrupt, match):
        p = tmp_path / "w.drwt"
        save_weights([np.zeros(2, np.float32)], p)
        d = bytearray(p.read_bytes())
        corrupt(d)
        p.write_bytes(bytes(d))
        with pytest.raises(ConfigError, match=match):
            load_weights(p)

    def test_truncated_and_trailing(self, tmp_path):
        p = tmp_path / "w.drwt"
        save_weights([np.zeros(4, np.float32)], p)
        p.write_bytes(p.read_bytes()[:-3])
        with pytest.raises(ConfigError, match="truncated"):
            load_weights(p)
        save_weights([np.zeros(4, np.float32)], p)
        p.write_bytes(p.read_bytes() + b"x")
        with pytest.raises(ConfigError, match="trailing"):
            load_weights(p)

    def test_parameter_layout_matches_reference_model(self):
        """72 tensors / 598,659 parameters for the default network."""
        specs = parameter_specs(DsttConfig())
        assert len(specs) == 72
        assert sum(int(np.prod(s)) for _, s in specs) == 598659
        w = seed_parameters(DsttConfig.baseline(64), 0)
        assert all(np.all(a == 0) for (n, _), a in zip(specs, w) if n.endswith("bias"))
        with pytest.raises(ConfigError):
            check_shapes(DsttConfig.baseline(64), w[:-1])


# ------------------------------------------------------------------ masks
def _diamond(k):
    return 2 * k * k + 2 * k + 1


class TestMasks:
    def test_redact_pixelwise(self, rng):
        rgb = rng.integers(0, 256, size=(24, 32, 3), dtype=np.uint8)
        mask = BinaryMask(rng.random((24, 32)) > 0.5)
        out = redact(rgb, mask)
        assert (out[mask.bits] == 0).all() and np.array_equal(out[~mask.bits], rgb[~mask.bits])
        assert np.array_equal(redact(out, mask), out)
        with pytest.raises(InputError):
            redact(rgb, BinaryMask.empty(8, 8))

    def test_adjust_area_grows_by_cross_diamond(self):
        bits = np.zeros((100, 100), bool)
        bits[50, 50] = True
        out = adjust_mask_area(BinaryMask(bits), 0.05, 0.30)
        k = next(k for k in range(100) if _diamond(k) >= 500)
        assert out.area() == _diamond(k)

    def test_adjust_area_erodes_and_fails(self):
        out = adjust_mask_area(BinaryMask.full(40, 40), 0.05, 0.30)
        x, y, w, h = out.tight_bbox()
        assert out.area_fraction() <= 0.30 and x == y and w == h and x > 0
        with pytest.raises(DegenerateMaskError):
            adjust_mask_area(BinaryMask.empty(10, 10), 0.05, 0.3)


# ------------------------------------------------------------------ synthetic inputs
def test_synthetic_generators_are_seeded_and_in_range():
    a, ma = synth.c2_frame(7, 128)
    b, mb = synth.c2_frame(7, 128)
    assert np.array_equal(a, b) and np.array_equal(ma, mb)
    assert a.dtype == np.float32 and 0.0 <= a.min() and a.max() <= 1.0
    assert 0.05 <= ma.mean() <= 0.30
    img, m = synth.c1_frame(0, 256)
    assert 0.10 <= m.mean() <= 0.26
    st = synth.C3Stream(0, 128, 10)
    f0, m0 = st.frame(0)
    f1, _ = st.frame(1)
    assert f0.shape == (3, 128, 128) and not np.array_equal(f0, f1)


# ------------------------------------------------------------------ C-ABI library
def _declared_functions():
    src = HEADER.read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dr_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_bound_interface():
    assert set(_declared_functions()) == set(_lib.SIGNATURES)


def test_library_loads_and_exports_every_declared_symbol():
    if not _lib.LIB_PATH.exists():
        pytest.skip("libdrb200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in _declared_functions():
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)],
                        capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dr_[a-z0-9_]+)\b", nm))
    assert set(_declared_functions()) <= exported
    assert _lib.load().dr_version() == 1


def test_struct_layouts_match_header():
    """ctypes mirrors of dr_config / dr_frame_io have the C sizes."""
    assert ctypes.sizeof(_lib.DrConfig) == 4 * 8 + 16 + 4 * 3
    assert ctypes.sizeof(_lib.DrFrameIO) == 8 * 16
    assert [f for f, _ in _lib.DrFrameIO._fields_][-1] == "slot_kv_reuse"


def test_error_codes_map_to_reference_exceptions():
    from paper_2509_10466_b200 import EngineNumericError
    assert _lib.DR_ERR_CONFIG == 1 and _lib.DR_ERR_INPUT == 2 and _lib.DR_ERR_NUMERIC == 3
    if _lib.LIB_PATH.exists():
        with pytest.raises(ConfigError):
            _lib.check(_lib.DR_ERR_CONFIG)
        with pytest.raises(InputError):
            _lib.check(_lib.DR_ERR_INPUT)
        with pytest.raises(EngineNumericError):
            _lib.check(_lib.DR_ERR_NUMERIC)


def test_engine_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2509_10466_b200 import DeviceError, DsttEngine
    with pytest.raises(DeviceError):
        DsttEngine(DsttConfig.baseline(64))


def test_batch_streamer_needs_a_gpu_and_is_exported():
    """The overlapped batch API is public and, like every compute entry point, raises
    instead of falling back to the CPU."""
    import paper_2509_10466_b200 as pkg
    from paper_2509_10466_b200.errors import DeviceError
    import torch
    assert "BatchStreamer" in pkg.__all__
    if torch.cuda.is_available():
        pytest.skip("GPU present: tests/test_gpu_streaming.py covers it")
    with pytest.raises(DeviceError):
        pkg.BatchStreamer(None, 2)
