"""Per-CTA timeline of the tcgen05 attention kernel (diagnostic build, -DDR_TRACE).

    python -m paper_2509_10466_b200.build --trace     # -> paper_2509_10466_b200/_build_trace/
    python scripts/attn_trace.py [--config C2]

Runs one un-graphed frame; for each attention launch of it prints the distribution over CTAs
of: start skew (entry - first entry), prologue (entry -> pdl_wait done), first S ready,
softmax loop, merge, and the kernel span, plus CTAs per SM.
"""

import argparse
import ctypes
import sys
from collections import Counter
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2509_10466_b200 import _lib  # noqa: E402

TRACE_LIB = _lib.LIB_PATH.parent.parent / "_build_trace" / _lib.LIB_PATH.name


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C2")
    args = p.parse_args()
    _lib.LIB_PATH = TRACE_LIB                      # must precede the first load()
    import torch

    import bench
    from paper_2509_10466_b200 import DsttEngine

    cfg, B, carried, _ = bench.workload(args.config)
    imgs, masks = bench.make_pool(args.config, B, 0, cfg.width)
    eng = DsttEngine(cfg, seed=0)
    img = torch.from_numpy(imgs).cuda()
    msk = torch.from_numpy(masks.astype(np.uint8)).cuda()
    mem = eng.zero_memory()
    eng.run(img, msk, mem.slots if carried else None)
    torch.cuda.synchronize()

    lib = _lib.load()
    fn = lib.dr_debug_attn_trace
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    n = 8192 * 16
    buf = (ctypes.c_ulonglong * n)()
    for idx in range(16):
        k = fn(idx, buf, n)
        if k <= 0:
            break
        t = np.frombuffer(buf, dtype=np.uint64, count=k).reshape(-1, 16).astype(np.int64)
        t0 = t[:, 0].min()
        rel = (t[:, :6] - t0) / 1000.0               # us
        span = rel[:, 5].max()
        pct = lambda v: "p0 %6.2f  p50 %6.2f  p100 %6.2f" % (v.min(), np.median(v), v.max())  # noqa
        print(f"launch {idx}: {len(t)} CTAs, span {span:.2f} us, blocks/CTA {Counter(t[:, 7])}")
        print("  entry skew      ", pct(rel[:, 0]))
        print("  prologue        ", pct(rel[:, 1] - rel[:, 0]))
        print("  first S ready   ", pct(rel[:, 2] - rel[:, 1]))
        print("  softmax loop    ", pct(rel[:, 3] - rel[:, 2]))
        rel8 = (t[:, 8:10] - t0) / 1000.0
        print("  O read (o_done) ", pct(rel8[:, 0] - rel[:, 3]))
        print("  DSMEM stores    ", pct(rel8[:, 1] - rel8[:, 0]))
        print("  cluster_sync    ", pct(rel[:, 4] - rel8[:, 1]))
        # cluster imbalance: loop-end spread within a cluster (key parts of one tile group)
        k = int(t[:, 10].max()) + 1
        if k > 1 and len(t) % k == 0:
            ends = rel[:, 3].reshape(-1, k)
            print("  cluster loop-end spread", pct(ends.max(1) - ends.min(1)))
        print("  tail            ", pct(rel[:, 5] - rel[:, 4]))
        print("  exit            ", pct(rel[:, 5]))
        per_sm = Counter(t[:, 6])
        print("  CTAs per SM     ", Counter(per_sm.values()), "SMs used", len(per_sm))
        # per-SM busy span: first entry to last exit
        loop = rel[:, 3] - rel[:, 2]
        sm = t[:, 6]
        for cnt in sorted(set(per_sm.values()), reverse=True):
            sms = [s for s, c in per_sm.items() if c == cnt]
            print(f"  loop on {cnt}-CTA SMs", pct(loop[np.isin(sm, sms)]))

if __name__ == "__main__":
    main()
