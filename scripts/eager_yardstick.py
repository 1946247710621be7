"""PyTorch-eager GPU yardstick: the reference's own DsttModel on cuda:0 (a measurement only,
never a bench arm).

    python scripts/eager_yardstick.py [--steps 20] > profiles/r02/eager_yardstick.json

Runs the UNMODIFIED reference model from baseline/_ref (dimreal, installed by
baseline/install_ref.sh; dstt.py:224-268) with `.cuda()`, in fp32 and under
torch.autocast(float16), on GPU-resident inputs:

* C2: 512x512, batch 1, memory carried frame to frame (dstt.py:309-311)
* C5: 512x512, batch 64 independent frames, cold (zero) memory

Timed per step with CUDA events: the network forward plus the fp32 alpha composite
(torch ops).  The mask stage (dilate + feather) is not included -- it has no GPU form in
the reference -- so the numbers are an upper bound on eager frames/s.  Prints one JSON
object per (config, precision).
"""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "baseline"))

import torch  # noqa: E402

import ref_path  # noqa: E402


def run(size, batch, carried, amp, steps, warmup):
    _, dstt = ref_path._import()
    cfg = dstt.DsttConfig(width=size, height=size, temporal_groups=4)
    model = dstt.DsttEngine(cfg, seed=0).model.cuda().eval()
    g = torch.Generator(device="cuda").manual_seed(0)
    rgb = torch.rand(batch, 3, size, size, device="cuda", generator=g)
    mask = (torch.rand(batch, 1, size, size, device="cuda", generator=g) < 0.15).float()
    rgb = rgb * (1 - mask)
    alpha = mask.clone()
    zero = torch.zeros(batch, cfg.tokens, cfg.channels, device="cuda")
    slots = (zero, zero)
    times = []
    with torch.no_grad(), torch.autocast("cuda", dtype=torch.float16, enabled=amp):
        for k in range(warmup + steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fill, new_slot = model(rgb, mask, slots)
            out = alpha * fill.float() + (1 - alpha) * rgb
            b.record()
            if carried:
                slots = (slots[1], new_slot)
            torch.cuda.synchronize()
            if k >= warmup:
                times.append(a.elapsed_time(b))
    del out
    times.sort()
    p50 = times[len(times) // 2]
    return {"config": "C2" if batch == 1 else "C5", "size": size, "batch": batch,
            "precision": "autocast_fp16" if amp else "fp32", "steps": steps,
            "ms_per_step_p50": round(p50, 3), "ms_per_step_min": round(times[0], 3),
            "frames_per_s": round(batch * 1000.0 / p50, 1),
            "note": "reference DsttModel eager on cuda:0; network + composite, no mask stage"}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    args = p.parse_args()
    why = ref_path.available()
    if why:
        print(json.dumps({"unavailable": why}))
        return
    print(json.dumps({"gpu": torch.cuda.get_device_name(0), "torch": torch.__version__}))
    for batch, carried in ((1, True), (64, False)):
        for amp in (False, True):
            steps = args.steps if batch == 1 else max(3, args.steps // 4)
            print(json.dumps(run(512, batch, carried, amp, steps, args.warmup)), flush=True)


if __name__ == "__main__":
    main()
