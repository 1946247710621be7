"""Fused decoder vs the unfused Vec2Patch -> decode.0 -> decode.2 path and the oracle
(diagnostic): max-abs of the raw network output at several sizes / batches.

    python scripts/dec_check.py
"""
import os
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2509_10466_b200 import DsttConfig, DsttEngine, synth
size, B, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
cfg = DsttConfig.baseline(size, mask_dilate=3, mask_feather_sigma=2.0)
eng = DsttEngine(cfg, seed=0)
imgs, masks = synth.frame_pool("C1", B, size=size)
rng = np.random.default_rng(1)
slots = [torch.from_numpy(rng.normal(0, 1, (B, cfg.tokens, 64)).astype(np.float32)).cuda() for _ in range(2)]
res = eng.run(torch.from_numpy(imgs).cuda(), torch.from_numpy(masks).cuda(), slots, want_fill=True)
np.savez(out, fill=res["fill"].cpu().numpy(), out=res["out"].cpu().numpy(), slot=res["slot"].cpu().numpy())
'''


def run(size, B, fused):
    dst = f"/tmp/dec_{size}_{B}_{fused}.npz"
    subprocess.run([sys.executable, "-c", CHILD, str(REPO), str(size), str(B), dst], check=True,
                   env={**os.environ, "DR_DEC_FUSED": str(fused)}, timeout=600)
    import numpy as np
    return np.load(dst)


def main():
    import numpy as np

    from oracle import dstt_oracle as O
    from paper_2509_10466_b200 import DsttConfig, synth
    from paper_2509_10466_b200.weights import seed_parameters
    for size, B in ((64, 2), (128, 1), (256, 1), (512, 1), (512, 5)):
        a, b = run(size, B, 1), run(size, B, 0)
        d = np.abs(a["fill"].astype(np.float64) - b["fill"])
        worst = np.unravel_index(np.argmax(d), d.shape)
        line = f"{size}^2 B={B}: fused vs unfused fill max-abs {d.max():.3e} at {worst}"
        if size <= 256:
            cfg = DsttConfig.baseline(size, mask_dilate=3, mask_feather_sigma=2.0)
            imgs, masks = synth.frame_pool("C1", B, size=size)
            rng = np.random.default_rng(1)
            slots = [rng.normal(0, 1, (B, cfg.tokens, 64)).astype(np.float32) for _ in range(2)]
            ref = O.inpaint_path(cfg, seed_parameters(cfg, 0), imgs, masks, slots)
            line += (f"; vs oracle fused {np.abs(a['fill'] - ref['fill']).max():.3e}"
                     f" unfused {np.abs(b['fill'] - ref['fill']).max():.3e}")
        print(line, flush=True)


if __name__ == "__main__":
    main()
