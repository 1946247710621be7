"""Per-CTA tile timeline of the tcgen05 conv kernels (diagnostic build, -DDR_TRACE).

    python -m paper_2509_10466_b200.build --trace
    python scripts/conv_trace.py

Runs one un-graphed C2 frame; for decode.0 and decode.2 prints, over CTAs and tiles, the
prologue (entry -> weights in smem), per-tile TMA latency (issue -> halo landed), MMA
issue span, accumulator wait (commit -> epilogue sees it), epilogue time, and the gaps
that show which stage paces the pipeline.
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2509_10466_b200 import _lib  # noqa: E402

TRACE_LIB = _lib.LIB_PATH.parent.parent / "_build_trace" / _lib.LIB_PATH.name


def pct(v):
    v = np.asarray(v, float)
    v = v[np.isfinite(v)]
    return "p10 %6.2f  p50 %6.2f  p90 %6.2f  max %6.2f" % tuple(np.percentile(v, [10, 50, 90, 100])) if v.size else "-"


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
    eng.run(img, msk, eng.zero_memory().slots)
    torch.cuda.synchronize()
    lib = _lib.load()
    fn = lib.dr_debug_conv_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    n = 256 * 128
    buf = (ctypes.c_ulonglong * n)()
    for idx, name in enumerate(["decode.0", "decode.2"]):
        k = fn(idx, buf, n)
        if k <= 0:
            break
        t = np.frombuffer(buf, dtype=np.uint64, count=k).reshape(-1, 128).astype(np.float64)
        t0 = t[:, :1]                       # per-CTA origin (clock64 is per SM)
        r = (t - t0) / 1965.0               # cycles -> us at 1965 MHz
        ntile = [int(((t[c, 3:83:5] > 0) & (t[c, 3:83:5] >= t[c, 0])).sum()) for c in range(len(t))]
        print(f"{name}: {len(t)} CTAs, span {r[:, 2].max():.2f} us, tiles/CTA {np.bincount(ntile)}")
        print("  weights landed    ", pct(r[:, 1] - r[:, 0]))
        tma, mma, accw, epi, gap_mma = [], [], [], [], []
        for c in range(len(t)):
            for i in range(ntile[c]):
                b = 3 + 5 * i
                tma.append(r[c, b + 1] - r[c, b])
                mma.append(r[c, b + 2] - r[c, b + 1])
                accw.append(r[c, b + 3] - r[c, b + 2])
                epi.append(r[c, b + 4] - r[c, b + 3])
                if i:
                    gap_mma.append(r[c, b + 1] - r[c, b - 5 + 2])   # halo landed - prev commit
        print("  TMA issue->landed ", pct(tma))
        print("  MMA issue span    ", pct(mma))
        print("  commit->epi sees  ", pct(accw))
        print("  epilogue          ", pct(epi))
        print("  prev commit->halo ", pct(gap_mma))
        last = [r[c, 3 + 5 * (ntile[c] - 1) + 4] for c in range(len(t)) if ntile[c]]
        print("  last epi done     ", pct(last), " exit", pct(r[:, 2]))




def dump_cta0():
    """Raw stamps of CTA 0 of decode.0 (debug)."""
    lib = _lib.load()
    fn = lib.dr_debug_conv_trace
    buf = (ctypes.c_ulonglong * (256 * 128))()
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    k = fn(0, buf, 256 * 128)
    t = np.frombuffer(buf, dtype=np.uint64, count=k).reshape(-1, 128).astype(np.int64)
    print("cta0", ((t[0, :45] - t[0, 0]) / 1965.0).round(2).tolist())


if __name__ == "__main__":
    main()
    dump_cta0()
