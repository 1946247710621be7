"""Per-CTA wait breakdown of the fused decoder (diagnostic build, -DDR_TRACE).

    python -m paper_2509_10466_b200.build --trace
    python scripts/dec_trace.py [--config C2]
"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2509_10466_b200 import _lib  # noqa: E402

NAMES = {2: "MMA wait w_full", 3: "MMA wait d_empty", 4: "E warp wait a2_full",
         5: "E warp wait e_empty", 6: "epi1 wait d_full", 8: "epi1 wait a2_empty",
         9: "epi2 wait e_full", 10: "epi2 phase barrier"}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C2")
    args = p.parse_args()
    import os
    _lib.LIB_PATH = _lib.LIB_PATH.parent.parent / os.environ.get("DEC_TRACE_BUILD", "_build_trace") / _lib.LIB_PATH.name
    import torch

    import bench
    from paper_2509_10466_b200 import DsttEngine
    cfg, B, carried, _ = bench.workload(args.config)
    imgs, masks = bench.make_pool(args.config, B, 0, cfg.width)
    eng = DsttEngine(cfg, seed=0)
    eng.run(torch.from_numpy(imgs).cuda(), torch.from_numpy(masks.astype(np.uint8)).cuda(), None)
    torch.cuda.synchronize()
    lib = _lib.load()
    fn = lib.dr_debug_dec_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    buf = (ctypes.c_ulonglong * (4096 * 16))()
    k = fn(0, buf, 4096 * 16)
    t = np.frombuffer(buf, dtype=np.uint64, count=k).reshape(-1, 16).astype(np.int64)
    t0 = t[:, 0].min()
    us = lambda c: c / 1965.0  # noqa: E731  cycles -> us
    pct = lambda v: "p0 %7.2f  p50 %7.2f  p100 %7.2f" % (v.min(), np.median(v), v.max())  # noqa
    print(f"{len(t)} CTAs")
    print("  start            ", pct((t[:, 0] - t0) / 1e3))
    print("  main loop (us)   ", pct((t[:, 12] - t[:, 0]) / 1e3))
    print("  finish pass (us) ", pct((t[:, 13] - t[:, 12]) / 1e3))
    print("   of which pixels", pct((t[:, 11] - t[:, 12]) / 1e3))
    tl = (ctypes.c_ulonglong * 384)()
    if fn(1, tl, 384) == 384:
        v = np.frombuffer(tl, dtype=np.uint64).reshape(6, 64).astype(np.int64)
        st = v[4, 0]
        print("  CTA 0 timeline (us from start): quad: MMA issue start / D committed / epi1 done / E committed / epi2 done")
        for i in range(16):
            print("    %2d: %7.2f %7.2f %7.2f %7.2f %7.2f" % ((i,) + tuple((v[k, i] - st) / 1965.0 for k in (5, 0, 1, 2, 3))))
    for s, n in NAMES.items():
        per_warp = 1 if s <= 5 else (4 if s >= 9 else 8)
        print(f"  {n:18s}", pct(us(t[:, s] / per_warp)))


if __name__ == "__main__":
    main()
