"""Per-CTA phase timeline of the Vec2Patch kernel (diagnostic build, -DDR_TRACE): one C2
frame; medians over CTAs (us at 1965 MHz, clock64 per SM)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2509_10466_b200 import _lib  # noqa: E402

TRACE_LIB = _lib.LIB_PATH.parent.parent / "_build_trace" / _lib.LIB_PATH.name


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
    for _ in range(2):
        eng.run(img, msk, eng.zero_memory().slots)
    torch.cuda.synchronize()
    fn = _lib.load().dr_debug_v2p_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    buf = (ctypes.c_ulonglong * (4096 * 20))()
    k = fn(buf, 4096 * 20)
    t = np.frombuffer(buf, dtype=np.uint64, count=k).reshape(-1, 20).astype(np.int64)
    t = t[t[:, 0] > 0][:280]
    r = (t - t[:, :1]) / 1965.0
    med = lambda v: f"{np.median(v):6.2f} (max {v.max():6.2f})"  # noqa: E731
    print(f"v2p: {len(t)} CTAs; CTA span {med(r[:, 19])} us")
    print(f"  alloc (pdl_wait)    {med(r[:, 1])}")
    print(f"  window landed       {med(r[:, 2])}")
    print("  MMA phase issued    " + " ".join(f"{np.median(r[:, 3 + p]):5.2f}" for p in range(8)))
    print("  epilogue phase done " + " ".join(f"{np.median(r[:, 11 + p]):5.2f}" for p in range(8)))


if __name__ == "__main__":
    main()
