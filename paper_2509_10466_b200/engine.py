"""The DSTT inpainting engine on B200: a drop-in for the reference `DsttEngine`.

Reference interfaces mirrored:
* `InpaintEngine` ABC and its template `inpaint()` (`inpaint/base.py:28-89`): width/height,
  zero_memory(), inpaint(rgb u8 HWC, BinaryMask, memory) -> EngineResult, same checks and
  exceptions (ConfigError / InputError / EngineNumericError), FIFO advanced once per call
  (also for empty masks), outside-mask pixels bit-exact.
* `DsttEngine(config, seed, weights_path)` (`inpaint/dstt.py:284-342`): seeded init
  (`_seed_parameters` :271-281), DRWT save/load (:328-342).
* `DsttModel.forward(rgb, mask, memory) -> (out, new_slot)` (`dstt.py:256-268`) as
  `model_forward`, batched on CUDA tensors; `forward` adds the mask stage and the alpha
  composite.

All compute runs in libdrb200.so (hand-written sm_100a kernels) behind the C-ABI of
`include/dr_b200.h`; there is no CPU fallback.  Memory slots are CUDA tensors, so the
FIFO advance is a pointer rotation.
"""

from __future__ import annotations

import ctypes
from abc import ABC, abstractmethod
from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import DsttConfig
from .errors import ConfigError, EngineNumericError, InputError
from .masks import BinaryMask
from .memory import InpaintMemory
from .weights import check_shapes, load_weights, save_weights, seed_parameters


@dataclass(frozen=True)
class EngineResult:
    rgb: np.ndarray            # (H, W, 3) uint8, same dims as input
    memory: InpaintMemory
    inference_ms: float


class InpaintEngine(ABC):
    """Fills masked regions of a redacted frame; carries two-slot memory (base.py:28-89)."""

    @property
    @abstractmethod
    def width(self) -> int: ...

    @property
    @abstractmethod
    def height(self) -> int: ...

    @abstractmethod
    def zero_memory(self) -> InpaintMemory: ...

    @abstractmethod
    def _fill(self, rgb, mask, memory): ...

    def _check_frame(self, rgb: np.ndarray, mask: BinaryMask) -> None:
        """base.py:60-67."""
        if rgb.shape != (self.height, self.width, 3):
            raise ConfigError(f"frame is {rgb.shape[1]}x{rgb.shape[0]}, engine expects "
                              f"{self.width}x{self.height}")
        if mask.bits.shape != rgb.shape[:2]:
            raise ConfigError("mask dimensions do not match engine resolution")
        if rgb.dtype != np.uint8:
            raise InputError("engine input must be an 8-bit rgb raster")


class _NativeEngine:
    """Owns one dr_engine* (weights repacked on the device)."""

    def __init__(self, cfg: DsttConfig, arrays, device: int):
        lib = _lib.load()
        arrays = [np.ascontiguousarray(a, dtype=np.float32) for a in arrays]
        n = len(arrays)
        ptrs = (ctypes.c_void_p * n)(*[a.ctypes.data for a in arrays])
        numels = (ctypes.c_int64 * n)(*[a.size for a in arrays])
        handle = ctypes.c_void_p()
        c = _lib.make_config(cfg)
        _lib.check(lib.dr_create(ctypes.byref(c), ptrs, numels, n, device, ctypes.byref(handle)))
        self.handle = handle
        self.lib = lib

    def close(self):
        if self.handle:
            self.lib.dr_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DsttEngine(InpaintEngine):
    """B200 engine with the reference DsttEngine surface.

    ``device``: CUDA device index.  Weights are seeded exactly like the reference
    (`seed_parameters`), or loaded from a DRWT file.
    """

    def __init__(self, config: DsttConfig | None = None, seed: int = 0, weights_path=None,
                 device: int = 0):
        torch = _lib.require_cuda()
        self.config = config or DsttConfig()
        self.device = torch.device("cuda", device)
        self._arrays = seed_parameters(self.config, seed)
        if weights_path is not None:
            self._arrays = check_shapes(self.config, load_weights(weights_path))
        self._native = _NativeEngine(self.config, self._arrays, device)
        self._flags = torch.zeros(64, dtype=torch.int32, device=self.device)

    @classmethod
    def from_arrays(cls, config: DsttConfig, arrays, device: int = 0) -> "DsttEngine":
        """Engine from explicit fp32 tensors in DRWT / state_dict order."""
        eng = cls.__new__(cls)
        torch = _lib.require_cuda()
        eng.config = config
        eng.device = torch.device("cuda", device)
        eng._arrays = check_shapes(config, arrays)
        eng._native = _NativeEngine(config, eng._arrays, device)
        eng._flags = torch.zeros(64, dtype=torch.int32, device=eng.device)
        return eng

    # ------------------------------------------------------------------ reference API
    @property
    def width(self) -> int:
        return self.config.width

    @property
    def height(self) -> int:
        return self.config.height

    @property
    def handle(self):
        return self._native.handle

    def zero_memory(self) -> InpaintMemory:
        """Cold memory (memory.py:32-34).  Both slots are one engine-held zero tensor; while
        it is unmodified (same storage, version counter unchanged) the launches receive
        it as the NULL zero slot, whose keys are a per-block constant (dr_b200.h)."""
        import torch
        z = self.__dict__.get("_zero")
        if z is None or z._version != self._zero_version:
            z = torch.zeros(self.config.tokens, self.config.channels, device=self.device)
            self._zero, self._zero_version = z, z._version
        return InpaintMemory.from_zero_slot(z)

    def _is_zero_slot(self, s) -> bool:
        import torch
        z = self.__dict__.get("_zero")
        return (z is not None and isinstance(s, torch.Tensor) and s.is_cuda
                and s.data_ptr() == z.data_ptr() and z._version == self._zero_version
                and s._version == self._zero_version and s.dtype == torch.float32
                and tuple(s.shape) in {tuple(z.shape), (1,) + tuple(z.shape)})

    def save_weights(self, path) -> None:
        save_weights(self._arrays, path)

    def load_weights(self, path) -> None:
        arrays = check_shapes(self.config, load_weights(path))
        native = _NativeEngine(self.config, arrays, self.device.index or 0)
        self._native.close()
        self._native, self._arrays = native, arrays

    def parameters(self) -> list[np.ndarray]:
        """The fp32 tensors in DRWT / state_dict order (host copies)."""
        return [a.copy() for a in self._arrays]

    def kernels_per_forward(self) -> int:
        return int(_lib.load().dr_kernels_per_forward(self.handle))

    def token_tile_rows(self, frames: int) -> int:
        """Tokens per CTA of the token-chain kernels at `frames` frames (128 = the
        throughput kernel with the last-block slot K/V fill)."""
        return int(_lib.load().dr_token_tile_rows(self.handle, frames))

    # Slot K/V cache bookkeeping (dr_frame_io.slot_kv_reuse): a memory slot may reuse the
    # K/V the engine computed when it produced that slot only if it is the very tensor the
    # engine wrote (same storage pointer, version counter unchanged = no in-place edits).
    def _register_slot(self, t) -> None:
        import weakref
        rec = (weakref.ref(t), t.data_ptr(), t._version, tuple(t.shape))
        self._produced = [r for r in getattr(self, "_produced", []) if r[0]() is not None][-5:]
        self._produced.append(rec)

    def _is_own_slot(self, s) -> bool:
        import torch
        if not isinstance(s, torch.Tensor) or not s.is_cuda or s.dtype != torch.float32:
            return False
        for ref, ptr, ver, shape in getattr(self, "_produced", []):
            t = ref()
            if t is None or ptr != s.data_ptr() or t._version != ver or s._version != ver:
                continue
            if tuple(s.shape) == shape or (len(shape) == 3 and shape[0] == 1
                                           and tuple(s.shape) == shape[1:]):
                return True
        return False

    def _slot(self, s):
        import torch
        if not isinstance(s, torch.Tensor):
            s = torch.as_tensor(np.asarray(s))
        return s.to(device=self.device, dtype=torch.float32).contiguous()

    def _fill(self, rgb, mask, memory):
        """Reference `_fill` contract: (filled u8 HWC, new slot, inference ms)."""
        import torch
        res = self.run(torch.from_numpy(np.ascontiguousarray(rgb))[None],
                       torch.from_numpy(mask.bits)[None], memory.slots, want_fill=True)
        fill = res["fill"][0].permute(1, 2, 0).mul(255.0).round().clamp(0, 255) \
            .to(torch.uint8).cpu().numpy()
        return fill, res["slot"][0], res["ms"]

    def inpaint(self, rgb: np.ndarray, mask: BinaryMask,
                memory: InpaintMemory | None = None) -> EngineResult:
        """InpaintEngine.inpaint (base.py:52-89): checks, the whole path on the device,
        the composite back in a new array, memory.push(new slot).  One C-ABI host call
        (dr_inpaint_u8_host_mem: pinned staging, one CUDA-graph launch, span-packed
        read-back) with the memory's slots passed explicitly."""
        import time

        import torch
        self._check_frame(rgb, mask)
        if memory is None:
            memory = self.zero_memory()
        T, C = self.config.tokens, self.config.channels
        slots = []
        for s in memory.slots:
            t = self._slot(s)
            if tuple(t.shape) == (1, T, C):
                t = t[0]
            if tuple(t.shape) != (T, C):
                raise ConfigError(f"memory slot shape {tuple(t.shape)} does not match tokens "
                                  f"({T}, {C})")
            slots.append(t)
        reuse = sum(1 << i for i, s in enumerate(memory.slots) if self._is_own_slot(s))
        ptrs = [0 if self._is_zero_slot(s) else t.data_ptr() for s, t in zip(memory.slots, slots)]
        new = self._fresh_slot(slots)
        bits = np.ascontiguousarray(mask.bits)
        if bits.dtype != np.uint8:
            bits = bits.astype(np.uint8) if bits.dtype != np.bool_ else bits.view(np.uint8)
        frame = np.ascontiguousarray(rgb)
        out = np.empty_like(frame)
        t0 = time.perf_counter()
        _lib.check(self._native.lib.dr_inpaint_u8_host_mem(
            self.handle, frame.ctypes.data, bits.ctypes.data, out.ctypes.data,
            ptrs[0], ptrs[1], new.data_ptr(), reuse,
            torch.cuda.current_stream(self.device).cuda_stream))
        ms = (time.perf_counter() - t0) * 1e3
        self._register_slot(new)
        return EngineResult(rgb=out, memory=memory.push(new), inference_ms=ms)

    def _fresh_slot(self, exclude):
        """A device [T][C] buffer for the next new slot.  Engine-owned buffers are recycled
        only when nothing outside the pool refers to them (no Python reference, no view of
        the storage), so memories a caller still holds are never overwritten; recycling
        keeps the host call's slot pointers, hence its CUDA graphs, to a few signatures."""
        import sys

        import torch
        pool = self.__dict__.setdefault("_slot_pool", [])
        busy = {t.data_ptr() for t in exclude}
        for i in range(len(pool)):
            t = pool[i]
            # references: the pool list, `t`, getrefcount's argument
            if (t.data_ptr() not in busy and sys.getrefcount(t) <= 3
                    and torch._C._storage_Use_Count(t.untyped_storage()._cdata) <= 2):
                return t
        t = torch.empty((self.config.tokens, self.config.channels), dtype=torch.float32,
                        device=self.device)
        if len(pool) < 8:
            pool.append(t)
        return t

    # ------------------------------------------------------------------ batched API
    def model_forward(self, rgb, mask, memory):
        """DsttModel.forward (dstt.py:256-268) on CUDA tensors: rgb (B,3,H,W) f32,
        mask (B,1,H,W) or (B,H,W), memory (slot0, slot1) each (T,C) or (B,T,C).
        Returns (out (B,3,H,W) f32 raw network output, new_slot (B,T,C))."""
        res = self.run(rgb, mask, memory, want_fill=True, composite=False)
        return res["fill"], res["slot"]

    def forward(self, rgb, mask, memory=None):
        """The whole hot path: mask stage -> forward -> alpha composite.
        Returns (composite (B,3,H,W) f32, new_slot (B,T,C))."""
        res = self.run(rgb, mask, memory)
        return res["out"], res["slot"]

    def run(self, rgb, mask, memory=None, *, want_fill=False, want_masks=False,
            composite=True, out=None, sync=True):
        """Launch the path once on the current stream.

        rgb: (B,3,H,W) f32 in [0,1] or (B,H,W,3) u8 (u8 API: u8 composite out, redaction
        checked).  mask: (B,H,W) / (B,1,H,W) bool/u8, nonzero = private.  Host tensors
        are copied to the device.  Returns a dict with "out", "slot", optionally "fill",
        "m1", "alpha", "token_valid", and "ms" (device time of the launch)."""
        torch = _lib.require_cuda()
        dev = self.device
        cfg = self.config
        u8 = rgb.dtype == torch.uint8
        if rgb.dim() != 4:
            raise ConfigError("rgb must be (B,3,H,W) f32 or (B,H,W,3) u8")
        B = rgb.shape[0]
        hw = tuple(rgb.shape[1:3]) if u8 else tuple(rgb.shape[-2:])
        if hw != (cfg.height, cfg.width):
            raise ConfigError(f"input is {hw[1]}x{hw[0]}, model is fixed at "
                              f"{cfg.width}x{cfg.height}")
        if u8 and rgb.shape[3] != 3 or (not u8 and rgb.shape[1] != 3):
            raise ConfigError("rgb must have 3 channels")
        rgb = rgb.to(device=dev, dtype=torch.uint8 if u8 else torch.float32,
                     non_blocking=True).contiguous()
        if mask.dim() == 4:
            mask = mask[:, 0]
        if tuple(mask.shape) != (B, cfg.height, cfg.width):
            raise ConfigError("mask dimensions do not match engine resolution")
        mask = mask.to(device=dev, non_blocking=True)
        mask = (mask != 0).to(torch.uint8) if mask.dtype != torch.uint8 else mask.contiguous()
        if memory is None:
            memory = self.zero_memory().slots
        reuse = sum(1 << i for i, s in enumerate(memory) if self._is_own_slot(s))
        zero = [self._is_zero_slot(s) for s in memory]
        slots = [self._slot(s) for s in memory]
        T, C = cfg.tokens, cfg.channels
        # the zero slot (passed as NULL) broadcasts to any batch
        shapes = {tuple(s.shape) for s, z in zip(slots, zero) if not z}
        if len(shapes) > 1:
            raise ConfigError("memory slots must share one shape")
        shape = shapes.pop() if shapes else tuple(slots[0].shape)
        if shape[-2:] != (T, C):
            raise ConfigError(f"memory slot shape {shape} does not match tokens ({T}, {C})")
        if len(shape) == 3 and shape[0] != B:
            if shape[0] == 1:
                slots = [s if z else s[0] for s, z in zip(slots, zero)]
                shape = shape[1:]
            else:
                raise ConfigError(f"memory slot batch {shape[0]} does not match {B} frames")
        batched = int(len(shape) == 3)
        o = out or {}
        new_slot = o.get("slot")
        if new_slot is None:
            new_slot = torch.empty((B, T, C), dtype=torch.float32, device=dev)
        res = {"slot": new_slot}
        io = _lib.DrFrameIO()
        io.frames = B
        io.mask_m0 = mask.data_ptr()
        io.slot0, io.slot1 = (0 if z else s.data_ptr() for z, s in zip(zero, slots))
        io.slot_batched = batched
        io.new_slot = new_slot.data_ptr()
        if u8:
            io.rgb_u8 = rgb.data_ptr()
            if composite:
                res["out"] = o.get("out") if o.get("out") is not None else \
                    torch.empty((B, cfg.height, cfg.width, 3), dtype=torch.uint8, device=dev)
                io.out_u8 = res["out"].data_ptr()
        else:
            io.rgb_f32 = rgb.data_ptr()
            if composite:
                res["out"] = o.get("out") if o.get("out") is not None else \
                    torch.empty((B, 3, cfg.height, cfg.width), dtype=torch.float32, device=dev)
                io.out_f32 = res["out"].data_ptr()
        if want_fill:
            res["fill"] = torch.empty((B, 3, cfg.height, cfg.width), dtype=torch.float32,
                                      device=dev)
            io.fill = res["fill"].data_ptr()
        if want_masks:
            res["m1"] = torch.empty((B, cfg.height, cfg.width), dtype=torch.uint8, device=dev)
            res["alpha"] = torch.empty((B, cfg.height, cfg.width), dtype=torch.float32,
                                       device=dev)
            res["token_valid"] = torch.empty((B, T), dtype=torch.uint8, device=dev)
            io.dilated = res["m1"].data_ptr()
            io.alpha = res["alpha"].data_ptr()
            io.token_valid = res["token_valid"].data_ptr()
        if self._flags.numel() < B:
            self._flags = torch.zeros(B, dtype=torch.int32, device=dev)
        fl = o.get("flags")                  # caller-owned int32 [>= B] flags words
        io.flags = (fl if fl is not None else self._flags).data_ptr()
        io.slot_kv_reuse = reuse
        stream = torch.cuda.current_stream(dev)
        if sync:
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
        _lib.check(self._native.lib.dr_forward(self.handle, ctypes.byref(io),
                                               stream.cuda_stream))
        self._register_slot(new_slot)
        # keep inputs alive until the launch is enqueued (ctypes holds raw pointers)
        res["_keep"] = (rgb, mask, slots)
        if sync:
            t1.record(stream)
            flags = self._flags[:B].cpu()        # synchronises the stream
            res["ms"] = t0.elapsed_time(t1)
            self._raise_flags(flags)
        return res

    @staticmethod
    def _raise_flags(flags) -> None:
        f = int(np.bitwise_or.reduce(flags.numpy().astype(np.int64))) if flags.numel() else 0
        if f & _lib.DR_FLAG_UNREDACTED:
            raise InputError("input is not redacted: nonzero pixels inside mask")
        if f & _lib.DR_FLAG_NONFINITE:
            raise EngineNumericError("model produced non-finite output")

    # ------------------------------------------------------------------ host buffers
    def inpaint_host(self, rgb: np.ndarray, mask_bits: np.ndarray) -> np.ndarray:
        """One u8 frame through host buffers (dr_inpaint_u8_host): the reference-facing
        C-ABI call, with the 2-slot memory held inside the engine."""
        torch = _lib.require_cuda()
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        if rgb.shape != (self.height, self.width, 3):
            raise ConfigError("frame does not match engine resolution")
        m = np.ascontiguousarray(mask_bits)
        if m.shape != (self.height, self.width):
            raise ConfigError("mask dimensions do not match engine resolution")
        m = m.view(np.uint8) if m.dtype == np.bool_ else np.ascontiguousarray(m, dtype=np.uint8)
        out = np.empty_like(rgb)
        _lib.check(self._native.lib.dr_inpaint_u8_host(
            self.handle, rgb.ctypes.data, m.ctypes.data, out.ctypes.data,
            torch.cuda.current_stream(self.device).cuda_stream))
        return out

    def reset_host_memory(self) -> None:
        _lib.check(self._native.lib.dr_reset_memory(self.handle))
