"""Per-CTA phase timeline of the tcgen05 token-chain kernels (diagnostic build, -DDR_TRACE).

    python -m paper_2509_10466_b200.build --trace
    python scripts/token_trace.py [--config C5]

One un-graphed frame batch (C2 default); for each token launch prints the median (over CTAs) time of every
phase between consecutive stamps of thread 0 (clock64, per SM; us at 1965 MHz).
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2509_10466_b200 import _lib  # noqa: E402

TRACE_LIB = _lib.LIB_PATH.parent.parent / "_build_trace" / _lib.LIB_PATH.name
NAMES = {0: "EMBED", 1: "POST", 2: "SLOTKV"}


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    args = ap.parse_args()
    _lib.LIB_PATH = TRACE_LIB
    import torch

    import bench
    from paper_2509_10466_b200 import DsttEngine
    cfg, B, carried, _ = bench.workload(args.config)
    imgs, masks = bench.make_pool(args.config, B, 0, cfg.width)
    eng = DsttEngine(cfg, seed=0)
    img = torch.from_numpy(imgs).cuda()
    msk = torch.from_numpy(masks.astype(np.uint8)).cuda()
    eng.run(img, msk, eng.zero_memory().slots)
    torch.cuda.synchronize()
    fn = _lib.load().dr_debug_tok_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    n = 1024 * 32 + 1
    buf = (ctypes.c_ulonglong * n)()
    for idx in range(16):
        k = fn(idx, buf, n)
        if k <= 0:
            break
        raw = np.frombuffer(buf, dtype=np.uint64, count=k).astype(np.int64)
        mode = int(raw[-1])
        t = raw[:-1].reshape(-1, 32)
        ok = t[:, 0] > 0
        t = t[ok]
        nst = int((t[0] > 0).sum())
        d = np.diff(t[:, :nst], axis=1) / 1965.0
        med = np.median(d, axis=0)
        tot = (t[:, nst - 1] - t[:, 0]) / 1965.0
        print(f"launch {idx} {NAMES.get(mode, mode)}: {len(t)} CTAs, CTA span p50 {np.median(tot):.2f} "
              f"max {tot.max():.2f} us; phases (p50 us): " + " ".join(f"{v:.2f}" for v in med))


if __name__ == "__main__":
    main()
