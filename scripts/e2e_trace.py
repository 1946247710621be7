"""Phase times of the host-buffer path (dr_inpaint_u8_host) on C2 frames, from the
engine's DR_E2E_TRACE instrumentation: host staging, enqueue, host fill, sync wait,
band copy-out, and the device-side H2D / forward / D2H spans (CUDA events).

    DR_E2E_TRACE=1 python scripts/e2e_trace.py
"""
import ctypes
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("DR_E2E_TRACE", "1")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2509_10466_b200 import DsttEngine, _lib  # noqa: E402

cfg, B, carried, _ = bench.workload("C2")
imgs, masks = bench.make_pool("C2", 8, 0, 512)
eng = DsttEngine(cfg, seed=0)
rgb8 = [np.ascontiguousarray(np.clip(np.rint(im.transpose(1, 2, 0) * 255), 0, 255).astype(np.uint8)) for im in imgs]
m8 = [np.ascontiguousarray(m.astype(np.uint8)) for m in masks]
for r, m in zip(rgb8, m8):
    r[m.astype(bool)] = 0
fn = _lib.load().dr_debug_e2e_trace
fn.argtypes = [ctypes.POINTER(ctypes.c_double)]
buf = (ctypes.c_double * 8)()
rows, walls = [], []
for i in range(600):
    t0 = time.perf_counter()
    eng.inpaint_host(rgb8[i % 8], m8[i % 8])
    walls.append((time.perf_counter() - t0) * 1e6)
    assert fn(buf) == 0
    if i >= 100:
        rows.append(list(buf))
a = np.median(np.array(rows), axis=0)
names = ["host staging in", "H2D+forward enqueue", "D2H enqueue+host fill", "sync wait",
         "band copy-out", "dev H2D", "dev forward", "dev D2H+flags"]
print(f"wall p50 {np.median(walls[100:]):.1f} us/frame (python call included)")
for n, v in zip(names, a):
    print(f"  {n:24s} {v:7.1f} us")
