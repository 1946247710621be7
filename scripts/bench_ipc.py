"""Frames/s of the C2 frame loop through the CUDA-IPC engine transport (service.py) vs the
in-process host-buffer path, both from host u8 frames (like the reference's
SocketEngineClient vs LocalEngineClient)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402


def factory():
    from paper_2509_10466_b200 import DsttConfig, DsttEngine
    return DsttEngine(DsttConfig.baseline(512, mask_dilate=5, mask_feather_sigma=3.0), seed=0)


def main():
    from paper_2509_10466_b200 import synth
    from paper_2509_10466_b200.service import IpcEngineServer
    frames = []
    for i in range(8):
        img, m = synth.c2_frame(i)
        rgb = np.ascontiguousarray(np.clip(np.rint(img.transpose(1, 2, 0) * 255), 0, 255).astype(np.uint8))
        rgb[m] = 0
        frames.append((rgb, m))
    srv = IpcEngineServer(factory).start()
    cli = srv.connect()
    for i in range(10):
        cli.inpaint_frame(i, *frames[i % 8])
    n = 300
    t0 = time.perf_counter()
    inf = 0.0
    for i in range(n):
        inf += cli.inpaint_frame(i, *frames[i % 8]).inference_ms
    dt = time.perf_counter() - t0
    cli.close()
    srv.stop()
    print(f"ipc transport: {n / dt:.1f} frames/s ({1e3 * dt / n:.3f} ms/frame, engine-side "
          f"{inf / n:.3f} ms)")
    eng = factory()
    eng.reset_host_memory()
    for i in range(10):
        eng.inpaint_host(*frames[i % 8])
    t0 = time.perf_counter()
    for i in range(n):
        eng.inpaint_host(*frames[i % 8])
    dt = time.perf_counter() - t0
    print(f"in-process host path: {n / dt:.1f} frames/s")


if __name__ == "__main__":
    main()
