"""Process-boundary transport for the engine over CUDA IPC.

The reference moves every frame through a local stream socket (DRIP, service.py:30-270:
`EngineServer(engine_factory)`, `SocketEngineClient.inpaint_frame`, one request in
flight, engine memory per connection).  Here the engine process exports three device
buffers once per connection (input rgb u8 HWC, mask u8, output u8 HWC) as CUDA IPC
handles (PyTorch's CUDA-tensor sharing = cudaIpcGetMemHandle / cudaIpcOpenMemHandle); per
frame the client copies its frame host->device straight into the engine's buffers, the
control pipe carries only (frame_id, op) and (status, inference_ms, message), and the
client reads the composite back from the shared output buffer.  No frame byte crosses the
socket, and the engine side never touches host memory (the paper's shared-device-memory
transport).

Surface mirrors the reference: `IpcEngineServer(engine_factory).start()`, `.connect()` ->
client with `inpaint_frame(frame_id, rgb, mask) -> InpaintCall`, `reset()`, `close()`,
`stop()`.  Engine errors come back as the reference exception classes.  Memory persists
across requests of a connection and resets on `reset()` / a new connection, like DRIP.
"""

from __future__ import annotations

import time
import traceback
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, EngineNumericError, InputError, ProtocolError

_ERRORS = {"ConfigError": ConfigError, "InputError": InputError,
           "EngineNumericError": EngineNumericError}


def _raise(name: str, message: str):
    if name == "ProtocolError":
        raise ProtocolError("op", message)
    raise _ERRORS.get(name, RuntimeError)(message)


@dataclass
class InpaintCall:
    """service.py:181-189."""
    rgb: np.ndarray
    inference_ms: float
    prep_ms: float
    transport_ms: float


def _serve(conn, engine_factory, device: str) -> None:
    """Engine process: owns the engine and the shared buffers, answers one request at a
    time until ('close',)."""
    import torch
    try:
        engine = engine_factory()
        h, w = engine.height, engine.width
        dev = torch.device(device)
        bufs = {"rgb": torch.zeros((h, w, 3), dtype=torch.uint8, device=dev),
                "mask": torch.zeros((h, w), dtype=torch.uint8, device=dev),
                "out": torch.zeros((h, w, 3), dtype=torch.uint8, device=dev)}
        conn.send(("ready", h, w, bufs))          # CUDA tensors travel as IPC handles
    except Exception as exc:                     # noqa: BLE001 -- reported to the client
        conn.send(("failed", type(exc).__name__, str(exc)))
        return
    memory = engine.zero_memory()
    while True:
        msg = conn.recv()
        op = msg[0]
        if op == "close":
            conn.send(("closed",))
            return
        if op == "reset":
            memory = engine.zero_memory()
            conn.send(("ok", 0.0))
            continue
        if op != "frame":
            conn.send(("err", "ProtocolError", f"unknown op {op!r}"))
            continue
        try:
            t0 = time.perf_counter()
            res = engine.run(bufs["rgb"][None], bufs["mask"][None], memory.slots,
                             out={"out": bufs["out"][None]})
            memory = memory.push(res["slot"][0])
            if device.startswith("cuda"):
                torch.cuda.synchronize(dev)
            conn.send(("ok", res.get("ms", 1e3 * (time.perf_counter() - t0))))
        except Exception as exc:                 # noqa: BLE001 -- mapped on the client
            conn.send(("err", type(exc).__name__, str(exc) or traceback.format_exc(limit=1)))


class IpcEngineClient:
    """`SocketEngineClient` surface (service.py:213-260) over the shared device buffers."""

    def __init__(self, conn, height: int, width: int, bufs, device: str):
        import torch
        self._conn = conn
        self.height, self.width = height, width
        self._bufs = bufs
        self._device = device
        pin = device.startswith("cuda")
        self._pin_rgb = torch.empty((height, width, 3), dtype=torch.uint8, pin_memory=pin)
        self._pin_mask = torch.empty((height, width), dtype=torch.uint8, pin_memory=pin)
        self._pin_out = torch.empty((height, width, 3), dtype=torch.uint8, pin_memory=pin)

    def _call(self, *msg):
        self._conn.send(msg)
        rep = self._conn.recv()
        if rep[0] == "err":
            _raise(rep[1], rep[2])
        return rep

    def inpaint_frame(self, frame_id: int, rgb: np.ndarray, mask) -> InpaintCall:
        import torch
        bits = np.asarray(getattr(mask, "bits", mask))
        if rgb.shape != (self.height, self.width, 3) or bits.shape != (self.height, self.width):
            raise ProtocolError("dimensions", f"frame {rgb.shape} / mask {bits.shape} vs "
                                              f"{self.width}x{self.height}")
        if rgb.dtype != np.uint8:
            raise InputError("engine input must be an 8-bit rgb raster")
        t0 = time.perf_counter()
        np.copyto(self._pin_rgb.numpy(), rgb)
        np.copyto(self._pin_mask.numpy(), bits, casting="unsafe")     # bool / u8 -> 0/1
        self._bufs["rgb"].copy_(self._pin_rgb, non_blocking=True)
        self._bufs["mask"].copy_(self._pin_mask, non_blocking=True)
        if self._device.startswith("cuda"):
            torch.cuda.current_stream().synchronize()   # frame is in the engine's memory
        t1 = time.perf_counter()
        rep = self._call("frame", int(frame_id))
        t2 = time.perf_counter()
        self._pin_out.copy_(self._bufs["out"])
        out = self._pin_out.numpy().copy()
        t3 = time.perf_counter()
        inference_ms = float(rep[1])
        return InpaintCall(rgb=out, inference_ms=inference_ms, prep_ms=1e3 * (t1 - t0),
                           transport_ms=max(0.0, 1e3 * ((t2 - t1) + (t3 - t2)) - inference_ms))

    def reset(self) -> None:
        self._call("reset")

    def close(self) -> None:
        if self._conn is not None:
            try:
                self._call("close")
            finally:
                self._conn.close()
                self._conn = None


class IpcEngineServer:
    """`EngineServer(engine_factory)` (service.py:154-178): one engine process per
    connection, built by `engine_factory` (a picklable callable) inside that process."""

    def __init__(self, engine_factory, device: str = "cuda"):
        self._factory = engine_factory
        self._device = device
        self._procs = []

    def start(self) -> "IpcEngineServer":
        return self

    def connect(self) -> IpcEngineClient:
        import torch.multiprocessing as mp
        ctx = mp.get_context("spawn")
        parent, child = ctx.Pipe()
        proc = ctx.Process(target=_serve, args=(child, self._factory, self._device), daemon=True)
        proc.start()
        self._procs.append(proc)
        rep = parent.recv()
        if rep[0] != "ready":
            proc.join(timeout=10)
            _raise(rep[1], rep[2])
        _, h, w, bufs = rep
        return IpcEngineClient(parent, h, w, bufs, self._device)

    def stop(self) -> None:
        for p in self._procs:
            p.join(timeout=10)
            if p.is_alive():
                p.terminate()
        self._procs = []
