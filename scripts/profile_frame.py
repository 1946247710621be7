"""Run N un-graphed frames of a BASELINE config through the engine (for ncu / sanitizer).

    python scripts/profile_frame.py [--config C2] [--frames 3]
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_10466_b200 import DsttEngine  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C2")
    p.add_argument("--frames", type=int, default=3)
    args = p.parse_args()
    cfg, B, carried, _ = bench.workload(args.config)
    imgs, masks = bench.make_pool(args.config, B, 0, cfg.width)
    eng = DsttEngine(cfg, seed=0)
    img = torch.from_numpy(imgs).cuda()
    msk = torch.from_numpy(masks.astype(np.uint8)).cuda()
    mem = eng.zero_memory()
    for _ in range(args.frames):
        res = eng.run(img, msk, mem.slots if carried else None)
        if carried:
            mem = mem.push(res["slot"][0])
    torch.cuda.synchronize()
    print(f"ok: {args.frames} frames of {args.config}, {eng.kernels_per_forward()} kernels each")


if __name__ == "__main__":
    main()
