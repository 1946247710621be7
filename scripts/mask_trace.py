"""Per-phase clock64 timeline of the fused mask stage (diagnostic build, -DDR_TRACE):
one C2 frame, median over the 256 CTAs of each phase (us at 1965 MHz)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2509_10466_b200 import _lib  # noqa: E402

TRACE_LIB = _lib.LIB_PATH.parent.parent / "_build_trace" / _lib.LIB_PATH.name
NAMES = ["pdl_wait", "loads (cp.async)", "m0->bits", "dilation", "col words", "vertical fp64",
         "nz mask", "horizontal fp64 + m1 out", "tokens + xin", "flags"]


def main():
    _lib.LIB_PATH = TRACE_LIB
    import torch

    import bench
    from paper_2509_10466_b200 import DsttEngine
    cfg, B, carried, _ = bench.workload("C2")
    imgs, masks = bench.make_pool("C2", B, 0, cfg.width)
    eng = DsttEngine(cfg, seed=0)
    img = torch.from_numpy(imgs).cuda()
    msk = torch.from_numpy(masks.astype(np.uint8)).cuda()
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    for _ in range(2):
        flush.zero_()
        eng.run(img, msk, eng.zero_memory().slots)
    torch.cuda.synchronize()
    fn = _lib.load().dr_debug_mask_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    n = 4096 * 16
    buf = (ctypes.c_ulonglong * n)()
    k = fn(buf, n)
    t = np.frombuffer(buf, dtype=np.uint64, count=k).reshape(-1, 16).astype(np.int64)[:256]
    d = np.diff(t[:, :10], axis=1) / 1965.0
    span = (t[:, 9] - t[:, 0]) / 1965.0
    print(f"mask stage: 256 CTAs, CTA span p50 {np.median(span):.2f} max {span.max():.2f} us")
    for i in range(9):
        print(f"  {NAMES[i]:28s} p50 {np.median(d[:, i]):6.2f}  max {d[:, i].max():6.2f} us")
    g0 = t[:, 11].min()
    start, end = (t[:, 11] - g0) / 1e3, (t[:, 12] - g0) / 1e3
    from collections import Counter
    per_sm = Counter(t[:, 13])
    print(f"  global: start p50 {np.median(start):.2f} max {start.max():.2f}, end p50 "
          f"{np.median(end):.2f} max {end.max():.2f} us; CTAs per SM {Counter(per_sm.values())}")
    order = np.argsort(-span)[:8]
    print("  slowest CTAs (block, span us, start us, SM, CTAs on SM):",
          [(int(b), round(float(span[b]), 2), round(float(start[b]), 2), int(t[b, 13]),
            per_sm[t[b, 13]]) for b in order])


if __name__ == "__main__":
    main()
