"""Batch inpainting from pinned host memory with the PCIe transfers overlapped.

`BatchStreamer` runs `DsttEngine.run` (the same forward, the same results) over a sequence
of u8 batches held in pinned host memory, with two device buffer sets alternating:

    upload stream    H2D rgb+mask of batch k+1 ----.
    compute stream   forward of batch k  -----------+--> flags word copied beside the output
    download stream  D2H composite + flags of batch k-1

so a batch's copies hide under its neighbours' compute (C5: 67 MB in and 50 MB out per
64-frame batch, ~2 ms of PCIe against a ~4.9 ms forward).  The forward reads only its own
buffer set, the download of a set finishes before the forward that overwrites it is
enqueued (host wait on an event two batches back), and per-stream memory stays on the
compute stream, so results equal the serial `run` bit for bit (tests/test_gpu_streaming.py).

There is no batched entry point in the reference (`InpaintEngine.inpaint`, base.py:52-89,
is one frame); this is the batch counterpart of the engine's host-buffer path for the
BASELINE batch configs (C3 streams, C5 offline batches).
"""

from __future__ import annotations

from . import _lib
from .errors import ConfigError


class BatchStreamer:
    """Overlapped batches through one engine.

    submit(rgb, mask, out, memory) enqueues one batch: rgb (B,H,W,3) u8 and mask (B,H,W)
    u8/bool in pinned host memory, out (B,H,W,3) u8 pinned host memory that receives the
    composite.  It returns the batch's new memory slot (device, (B,T,C)) for carried
    memory (with carry_memory=True the streamer keeps the 2-slot FIFO per stream itself,
    `memory` stays None, and the returned slot is valid for the next two submits).  Batch
    k's `out` is complete (and its redaction / non-finite flags checked) once
    submit() of batch k+2 has returned, or after finish(); a caller that reads the results
    rotates three `out` buffers (batch k+3 may reuse batch k's)."""

    # carry_memory: steady-state forwards as CUDA graph replays, one per (buffer set,
    # memory-ring phase): period lcm(2, 3) = 6, captured after GRAPH_WARM eager batches
    GRAPH_WARM = 6

    def __init__(self, engine, batch: int, carry_memory: bool = False, graphs: bool = True):
        torch = _lib.require_cuda()
        cfg = engine.config
        dev = engine.device
        self.engine, self.batch = engine, batch
        H, W = cfg.height, cfg.width
        self.d_rgb = [torch.empty((batch, H, W, 3), dtype=torch.uint8, device=dev) for _ in range(2)]
        self.d_mask = [torch.empty((batch, H, W), dtype=torch.uint8, device=dev) for _ in range(2)]
        self.d_out = [torch.empty((batch, H, W, 3), dtype=torch.uint8, device=dev) for _ in range(2)]
        self.d_flags = [torch.zeros(batch, dtype=torch.int32, device=dev) for _ in range(2)]
        self.h_flags = [torch.zeros(batch, dtype=torch.int32).pin_memory() for _ in range(2)]
        self.up = torch.cuda.Stream(dev)
        self.comp = torch.cuda.Stream(dev)
        self.down = torch.cuda.Stream(dev)
        self.ev_comp = [torch.cuda.Event() for _ in range(2)]
        self.ev_up = [torch.cuda.Event() for _ in range(2)]
        self.ev_down = [torch.cuda.Event() for _ in range(2)]
        self.pending = [False, False]
        self.k = 0
        self.own, self.own_refs = set(), []    # slots made on the compute stream (kept alive
                                               # so their ids stay unique)
        # carry_memory: the streamer holds each stream's 2-slot FIFO itself (like the
        # engine-held memory of dr_inpaint_u8_host): batch k reads the slots of batches k-2
        # and k-1 (zero slots before), writes ring[k % 3]
        self.carry = carry_memory
        self.graphs = {} if (carry_memory and graphs) else None
        if carry_memory:
            self.ring = [torch.zeros((batch, cfg.tokens, cfg.channels), dtype=torch.float32,
                                     device=dev) for _ in range(3)]

    def submit(self, rgb, mask, out, memory=None):
        torch = _lib.require_cuda()
        B = self.batch
        if tuple(rgb.shape) != tuple(self.d_rgb[0].shape) or rgb.dtype != torch.uint8:
            raise ConfigError(f"rgb must be u8 {tuple(self.d_rgb[0].shape)}")
        if tuple(mask.shape) != tuple(self.d_mask[0].shape):
            raise ConfigError(f"mask must be {tuple(self.d_mask[0].shape)}")
        if tuple(out.shape) != tuple(self.d_out[0].shape) or out.dtype != torch.uint8:
            raise ConfigError(f"out must be u8 {tuple(self.d_out[0].shape)}")
        i = self.k & 1
        if self.carry:
            if memory is not None:
                raise ConfigError("a carry_memory streamer holds the memory itself")
            k = self.k
            zero = self.engine.zero_memory().slots[0]
            memory = (zero if k < 2 else self.ring[(k - 2) % 3],
                      zero if k < 1 else self.ring[(k - 1) % 3])
        self._complete(i)                  # set i's last download done, its flags checked
        with torch.cuda.stream(self.up):
            self.d_rgb[i].copy_(rgb, non_blocking=True)
            self.d_mask[i].copy_(mask.view(torch.uint8) if mask.dtype == torch.bool else mask,
                                 non_blocking=True)
            self.ev_up[i].record(self.up)
        self.comp.wait_event(self.ev_up[i])
        # memory not made by this streamer (e.g. a zero slot on the caller's stream) is
        # complete before the forward reads it, and stays allocated until it is done
        foreign = [t for t in (memory or ()) if isinstance(t, torch.Tensor) and t.is_cuda
                   and id(t) not in self.own]
        if foreign:
            self.comp.wait_stream(torch.cuda.current_stream(self.engine.device))
            for t in foreign:
                t.record_stream(self.comp)
        outs = {"out": self.d_out[i], "flags": self.d_flags[i]}
        if self.carry:
            outs["slot"] = self.ring[self.k % 3]
        if self.graphs is not None and self.k >= self.GRAPH_WARM:
            # steady state: every launch decision (slot K/V cache entries included) repeats
            # with period 6, so the captured forward of phase k % 6 is replayed
            g = self.graphs.get(self.k % 6)
            if g is None:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.comp):
                    self.engine.run(self.d_rgb[i], self.d_mask[i], memory, sync=False, out=outs)
                self.graphs[self.k % 6] = g
            with torch.cuda.stream(self.comp):
                g.replay()
                self.ev_comp[i].record(self.comp)
            slot = outs["slot"]
        else:
            with torch.cuda.stream(self.comp):
                r = self.engine.run(self.d_rgb[i], self.d_mask[i], memory, sync=False, out=outs)
                self.ev_comp[i].record(self.comp)
            slot = r["slot"]
        self.own = {id(t) for t in (memory or ()) if id(t) in self.own} | {id(slot)}
        self.own_refs = [t for t in (memory or ()) if id(t) in self.own] + [slot]
        with torch.cuda.stream(self.down):
            self.down.wait_event(self.ev_comp[i])
            out.copy_(self.d_out[i], non_blocking=True)
            self.h_flags[i].copy_(self.d_flags[i], non_blocking=True)
            self.ev_down[i].record(self.down)
        self.pending[i] = True
        self.k += 1
        return slot

    def _complete(self, i: int) -> None:
        if self.pending[i]:
            self.ev_down[i].synchronize()
            self.pending[i] = False
            self.engine._raise_flags(self.h_flags[i])

    def finish(self) -> None:
        """Wait for every submitted batch; raises the first batch error found."""
        for i in (self.k & 1, (self.k + 1) & 1):
            self._complete(i)
