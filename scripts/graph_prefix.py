"""In-graph cost of each kernel of a C2 frame: CUDA-graph replays of the first k launches
(DR_STOP_AFTER=k, diagnostics only), device time per replay with CUDA events, L2 flushed
between replays like bench.py.  Prints k, the kernel added, prefix time, increment."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

NAMES13 = ["mask", "embed+qkv", "attn S", "post", "attn T", "post", "attn S", "post", "attn T",
           "post(last)", "vec2patch", "decode.0", "decode.2+composite"]
NAMES = NAMES13                      # replaced by the 15-launch list when slot K/V run


def time_prefix(k, reps=200):
    os.environ["DR_STOP_AFTER"] = str(k)
    from paper_2509_10466_b200 import DsttEngine
    cfg, B, carried, _ = bench.workload("C2")
    imgs, masks = bench.make_pool("C2", 2, 0, cfg.width)
    eng = DsttEngine(cfg, seed=0)
    img = torch.from_numpy(imgs[:1]).cuda()
    msk = torch.from_numpy(masks[:1].astype(np.uint8)).cuda()
    T = cfg.tokens
    ring = [torch.zeros((1, T, 64), device="cuda") for _ in range(3)]
    out = torch.empty((1, 3, 512, 512), device="cuda")
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):                                # warm: slot K/V cache in steady state
            eng.run(img, msk, (ring[0], ring[1]), out={"out": out, "slot": ring[2]}, sync=False)
            ring = [ring[1], ring[2], ring[0]]
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            eng.run(img, msk, (ring[0], ring[1]), out={"out": out, "slot": ring[2]}, sync=False)
        KERNELS[0] = eng.kernels_per_forward()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


KERNELS = [0]


def main():
    global NAMES
    prev = 0.0
    full = time_prefix(99)
    if KERNELS[0] == 15:
        NAMES = NAMES13[:1] + ["slot K/V", "slot K/V"] + NAMES13[1:]
    print(f"{KERNELS[0]} kernels per captured forward, full graph {full:.2f} us")
    for k in range(1, len(NAMES) + 1):
        t = time_prefix(k)
        print(f"k={k:2d} +{NAMES[k-1]:20s} prefix {t:7.2f} us  increment {t - prev:6.2f} us", flush=True)
        prev = t


if __name__ == "__main__":
    main()
