"""Where the host-buffer (e2e) frame time goes: C2 frames through dr_inpaint_u8_host vs
its parts (pinned staging copies, H2D/D2H, un-graphed forward, graphed forward)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_10466_b200 import DsttEngine  # noqa: E402


def t(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


cfg, B, carried, _ = bench.workload("C2")
imgs, masks = bench.make_pool("C2", 4, 0, 512)
eng = DsttEngine(cfg, seed=0)
rgb8 = [np.ascontiguousarray(np.clip(np.rint(im.transpose(1, 2, 0) * 255), 0, 255).astype(np.uint8)) for im in imgs]
m8 = [np.ascontiguousarray(m.astype(np.uint8)) for m in masks]
for r, m in zip(rgb8, m8):
    r[m.astype(bool)] = 0
k = [0]


def host():
    k[0] += 1
    eng.inpaint_host(rgb8[k[0] % 4], m8[k[0] % 4])


pin_in = torch.empty(512 * 512 * 4, dtype=torch.uint8).pin_memory()
pin_out = torch.empty(512 * 512 * 3, dtype=torch.uint8).pin_memory()
dev_in = torch.empty(512 * 512 * 4, dtype=torch.uint8, device="cuda")
dev_out = torch.empty(512 * 512 * 3, dtype=torch.uint8, device="cuda")
src = np.concatenate([rgb8[0].ravel(), m8[0].ravel()])
dst = np.empty(512 * 512 * 3, np.uint8)


def staging():
    pin_in.numpy()[:] = src
    dst[:] = pin_out.numpy()


def copies():
    dev_in.copy_(pin_in, non_blocking=True)
    pin_out.copy_(dev_out, non_blocking=True)
    torch.cuda.synchronize()


d_img = torch.from_numpy(imgs).cuda()
d_m = torch.from_numpy(masks.astype(np.uint8)).cuda()
mem = eng.zero_memory()


def fwd():
    res = eng.run(d_img[:1], d_m[:1], mem.slots, sync=False)


print(f"inpaint_host   {t(host):8.1f} us/frame")
print(f"staging memcpy {t(staging):8.1f} us (1.25 MB in + 0.75 MB out, numpy)")
print(f"H2D+D2H+sync   {t(copies):8.1f} us")
print(f"forward (eager launches, async) {t(fwd):8.1f} us")
