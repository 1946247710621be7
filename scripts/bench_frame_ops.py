"""Device timing of the frame byte kernels with achieved HBM GB/s.

    python scripts/bench_frame_ops.py [--h 720 --w 1280] [--iters 200]

Display composite at the reference's display path (capture H x W -> 2H x 2W, ~20 % mask),
merge + redact of 4 track masks, point-cloud transplant (60 % valid depth).  Algorithmic
bytes per launch are the compulsory reads + writes; CUDA events on the launch stream
around a CUDA graph of `iters` back-to-back launches (inputs L2-resident after the first:
the figure is the per-launch cost in the frame loop, where the producer just wrote them).
Prints one JSON line per op.
"""

import argparse
import json
import sys
from pathlib import Path
from types import SimpleNamespace

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_10466_b200 import _lib  # noqa: E402


def timed(fn, iters):
    """Mean device time per launch: `iters` launches captured in one CUDA graph (the ctypes
    call overhead would otherwise dominate these few-microsecond kernels), replayed
    between two CUDA events on the capture stream."""
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(iters):
                fn()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--h", type=int, default=720)
    p.add_argument("--w", type=int, default=1280)
    p.add_argument("--iters", type=int, default=200)
    args = p.parse_args()
    h, w = args.h, args.w
    rng = np.random.default_rng(0)
    dev = torch.device("cuda")
    lib = _lib.load()
    cur = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731 (the capture stream)
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
        if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0}
    orig = torch.from_numpy(rng.integers(0, 256, (h, w, 3), dtype=np.uint8)).to(dev)
    inp = torch.from_numpy(rng.integers(0, 256, (h, w, 3), dtype=np.uint8)).to(dev)
    yy, xx = np.mgrid[0:h, 0:w]
    mask_np = ((yy - h / 2) ** 2 / (0.3 * h) ** 2 + (xx - w / 2) ** 2 / (0.3 * w) ** 2 < 1)
    mask = torch.from_numpy(mask_np.astype(np.uint8)).to(dev)
    out = torch.empty((2 * h, 2 * w, 3), dtype=torch.uint8, device=dev)
    ms = timed(lambda: _lib.check(lib.dr_display_composite(h, w, 3, orig.data_ptr(), inp.data_ptr(),
                                                           mask.data_ptr(), 0, out.data_ptr(), cur())),
               args.iters)
    byts = h * w * (3 + 1) + int(mask_np.sum()) * 3 + 4 * h * w * 3
    rows = [("display_composite", ms, byts, f"{h}x{w} -> {2*h}x{2*w}, mask {mask_np.mean():.2f}")]

    masks = torch.from_numpy((rng.random((4, h, w)) > 0.8).astype(np.uint8)).to(dev)
    flags = torch.tensor([1, 0, 1, 1], dtype=torch.uint8, device=dev)
    merged = torch.empty((h, w), dtype=torch.uint8, device=dev)
    red = torch.empty_like(orig)
    ms = timed(lambda: _lib.check(lib.dr_merge_redact(4, h, w, masks.data_ptr(), flags.data_ptr(),
                                                      orig.data_ptr(), merged.data_ptr(),
                                                      red.data_ptr(), cur())), args.iters)
    rows.append(("merge_redact", ms, h * w * (3 + 3 + 1) + 3 * h * w, "4 track masks (3 private)"))

    depth_np = (rng.random((h, w)) * 4).astype(np.float32)
    depth_np[rng.random((h, w)) < 0.4] = 0
    depth = torch.from_numpy(depth_np).to(dev)
    xyz = torch.empty((h * w, 3), dtype=torch.float32, device=dev)
    col = torch.empty((h * w, 3), dtype=torch.uint8, device=dev)
    scratch = torch.empty(h + 1, dtype=torch.int32, device=dev)
    intr = SimpleNamespace(fx=900.0, fy=900.0, cx=w / 2, cy=h / 2)
    ms = timed(lambda: _lib.check(lib.dr_pack_pointcloud(h, w, depth.data_ptr(), inp.data_ptr(),
                                                         intr.fx, intr.fy, intr.cx, intr.cy,
                                                         scratch.data_ptr(), xyz.data_ptr(),
                                                         col.data_ptr(), scratch[h:].data_ptr(), cur())),
               args.iters)
    nv = int((depth_np > 0).sum())
    rows.append(("pack_pointcloud", ms, h * w * (4 + 3) + nv * 15, f"{nv} points (60% valid), 2 launches"))
    for name, ms, byts, note in rows:
        gbs = byts / (ms * 1e-3) / 1e9
        print(json.dumps({"op": name, "us_per_launch": round(ms * 1e3, 2), "alg_bytes": byts,
                          "achieved_gbs": round(gbs, 1), "hbm_peak_gbs": peak["hbm_gbs"],
                          "frac": round(gbs / peak["hbm_gbs"], 4), "note": note}))


if __name__ == "__main__":
    main()
