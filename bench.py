#!/usr/bin/env python
"""Benchmark of the B200 masked-inpainting hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2|C1|C4|C5]

Default workload = BASELINE configs[1] (C2): batch-1 real-time path at 512x512, the
reference network (patch 8, C 64, 4 heads, S,T,S,T, temporal_groups 4) with seeded
random-init weights (seed 0), dilation r=5, feather sigma=3, memory carried across
frames, seeded synthetic frames (blurred-uniform image + ellipse/brush mask).  One step =
one frame through mask stage -> forward -> composite.

value     frames/s over all ranks, device time: CUDA events around every step (a CUDA
          graph replay of the whole path), L2 flushed (256 MiB write) between steps
          outside the events, inputs resident in HBM; p50/p99 per-frame latency alongside.
e2e       frames/s through the reference-facing C-ABI call with HOST buffers
          (dr_inpaint_u8_host: u8 frame + mask in, u8 composite out, per frame).
roofline  dominant kernel class from live per-stage CUDA events (un-graphed profiled
          pass over the same frames), algorithmic FLOPs per launch / mean duration.
cpu_baseline  the CPU oracle port (numpy, oracle/dstt_oracle.py) on this host, rank 0.

--impl reference: the reference's CPU path (the oracle port; the reference is Python and
cannot be compiled or installed as a GPU arm) on the same config, rank 0 only.
N>1 (torchrun): one process per GPU, independent frames per rank (weak scaling), no
collective on the data path; barrier + max-over-ranks timing.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    p.add_argument("--pool", type=int, default=8, help="distinct seeded frames per rank")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    return p.parse_args()


# ---------------------------------------------------------------------------- workload
C3_STREAMS = 8


def workload(name, world=1):
    from paper_2509_10466_b200 import DsttConfig
    size = {"C1": 256, "C2": 512, "C3": 512, "C4": 1024, "C5": 512}[name]
    cfg = DsttConfig.baseline(size, mask_dilate=5, mask_feather_sigma=3.0,
                              mask_aware_attention=(name == "C4"))
    # C3: stream s runs on GPU s mod n; the co-resident streams of a GPU are one batch
    # with per-stream memory slots ([B][T][C])
    batch = {"C5": 64, "C3": max(1, C3_STREAMS // world)}.get(name, 1)
    carried = name in ("C1", "C2", "C3", "C4")
    desc = {"C1": "C1: 1x3x256^2 single frame, r=5, sigma=3",
            "C2": "C2: batch-1 real-time 1x3x512^2, r=5, sigma=3, memory carried",
            "C3": f"C3: {C3_STREAMS} video streams 3x512^2 (translating canvas, jittering "
                  "ellipse), streams batched per GPU with per-stream memory",
            "C4": "C4: 1x3x1024^2, 30-45% occlusion, mask-aware attention",
            "C5": "C5: batch 64 x 3x512^2 independent frames (cold memory)"}[name]
    return cfg, batch, carried, desc


def stage_flops(cfg):
    """Dense algorithmic FLOPs per frame of each kernel class (per launch)."""
    T, C, H, W = cfg.tokens, cfg.channels, cfg.height, cfg.width
    g = cfg.temporal_groups
    tg = T // g
    dh = C // cfg.heads
    qkv = 2 * T * C * 3 * C
    return {
        "embed_qkv": 2 * T * (4 * cfg.patch ** 2) * C + qkv,
        "slot_kv": 2 * T * C * 2 * C,
        "attn_spatial": 2 * 2 * cfg.heads * T * T * dh,
        "attn_temporal": 2 * 2 * cfg.heads * g * tg * (3 * tg) * dh,
        "mlp_qkv": 2 * T * (C * C + C * 2 * C + 2 * C * C) + qkv,
        "vec2patch": 2 * T * C * C * cfg.kernel ** 2,
        "decode0": 2 * H * W * C * C * 9,
        "decode2_composite": 2 * H * W * C * 3 * 9,
        "mask_stage": 0,
    }


def stage_exps(cfg):
    """Softmax exponentials per frame per attention launch (dense, all keys)."""
    T, g = cfg.tokens, cfg.temporal_groups
    tg = T // g
    return {"attn_spatial": cfg.heads * T * T, "attn_temporal": cfg.heads * g * tg * 3 * tg}


def frame_flops_reference(cfg):
    """Reference FlopCounterMode count per frame: the forward's dense
    contractions; attention counts QK^T and PV, linear layers once."""
    f = stage_flops(cfg)
    T, C = cfg.tokens, cfg.channels
    n_s = sum(b == "S" for b in cfg.blocks)
    n_t = len(cfg.blocks) - n_s
    per_block_lin = 2 * T * (4 * C * C + 4 * C * C)     # q,k,v,out + ffn (64x128 x2)
    t_extra = 2 * 2 * T * 2 * C * C                     # k,v over both slots
    return (2 * T * 4 * cfg.patch ** 2 * C + len(cfg.blocks) * per_block_lin
            + n_s * f["attn_spatial"] + n_t * (f["attn_temporal"] + t_extra)
            + f["vec2patch"] + f["decode0"] + f["decode2_composite"])


def make_pool(name, n, rank, size, world=1):
    from paper_2509_10466_b200 import synth
    if name == "C3":                       # n = frames x streams of this rank, time-major
        streams = [s for s in range(C3_STREAMS) if s % world == rank]
        src = [synth.C3Stream(s, size) for s in streams]
        imgs, masks = [], []
        for t in range(n // len(src)):
            for st in src:
                img, m = st.frame(t)
                imgs.append(img)
                masks.append(m)
        return np.stack(imgs), np.stack(masks)
    gen = {"C1": synth.c1_frame, "C2": synth.c2_frame, "C4": synth.c4_frame,
           "C5": synth.c5_frame}[name]
    imgs, masks = [], []
    for i in range(n):
        img, m = gen(rank * 100003 + i, size)
        imgs.append(img)
        masks.append(m)
    return np.stack(imgs), np.stack(masks)


def traffic(stage, batch):
    """DRAM bytes per launch of `stage` from the committed ncu capture (batch-1 C2 frames,
    scripts/ncu_traffic.py), or None when there is no capture for this workload."""
    p = REPO / "profiles" / "r01" / "ncu_traffic.json"
    if batch != 1 or not p.exists():
        return None
    st = json.loads(p.read_text())["stages"].get(stage)
    return None if st is None else round(st["dram_bytes_per_launch"])


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return dict(FALLBACK_PEAKS), "fallback"


# ---------------------------------------------------------------------------- clocks
class Clocks:
    """SM clock + throttle-reason sampler running DURING the timed region: an NVML thread
    polling every ~2 ms (the batch-1 timed region is tens of ms, too short for the
    100 ms floor of `nvidia-smi -lms`); falls back to one nvidia-smi query."""
    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index, period_s=0.002):
        import threading
        self.rows, self.max_mhz, self.nvml = [], None, None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.nvml = (pynvml, h)
        except Exception:
            self.nvml = None
        self.index = index
        self.stop_ev = threading.Event()
        self.thread = threading.Thread(target=self._run, args=(period_s,), daemon=True)
        self.thread.start()

    def _run(self, period_s):
        if self.nvml is None:
            return
        pynvml, h = self.nvml
        bits = {k: getattr(pynvml, v, 0) for k, v in self.REASONS.items()}
        while not self.stop_ev.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), {k for k, b in bits.items() if rs & b}))
            except Exception:
                pass
            self.stop_ev.wait(period_s)

    def stop(self):
        self.stop_ev.set()
        self.thread.join(timeout=5)
        if not self.rows:
            try:
                q = subprocess.run(["nvidia-smi", f"--id={self.index}",
                                    "--query-gpu=clocks.sm,clocks.max.sm",
                                    "--format=csv,noheader,nounits"],
                                   capture_output=True, text=True, timeout=10).stdout.split(",")
                return {"sm_mhz": float(q[0]), "sm_max_mhz": float(q[1]), "samples": 1,
                        "reasons": [], "source": "nvidia-smi after the timed region"}
            except Exception:
                return None
        sm = [r[0] for r in self.rows]
        reasons = sorted(set().union(*(r[1] for r in self.rows)))
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm),
                "sm_max_mhz": self.max_mhz, "samples": len(self.rows), "reasons": reasons,
                "source": "NVML every 2 ms during the timed region"}


# ---------------------------------------------------------------------------- CPU arm
def cpu_oracle_rate(name, seconds, max_frames=64):
    """The CPU oracle (numpy port of the reference path) on this host: frames/s over a
    bounded sample of the workload, memory carried for the streaming configs."""
    from oracle import dstt_oracle as O
    from paper_2509_10466_b200 import synth
    from paper_2509_10466_b200.weights import seed_parameters
    cfg, batch, carried, _ = workload(name)
    size = cfg.width
    w = O.Params(cfg, seed_parameters(cfg, 0))
    zero = np.zeros((cfg.tokens, cfg.channels), np.float32)
    slots = (zero, zero)
    t0 = time.perf_counter()
    n = 0
    while True:
        if name == "C3":
            img, m = synth.C3Stream(0, size).frame(n)
            img, m = img[None], m[None]
        else:
            img, m = make_pool(name, 1, 0, size) if name != "C2" else _c2(n)
        res = O.inpaint_path(cfg, w, img, m, slots)
        if carried:
            slots = (slots[1], res["slot"][0])
        n += 1
        el = time.perf_counter() - t0
        if (el >= seconds and n >= 2) or n >= max_frames:
            break
    return n / el, n, el


def _c2(seed):
    from paper_2509_10466_b200 import synth
    img, m = synth.c2_frame(seed)
    return img[None], m[None]


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, batch, carried, desc = workload(args.config)
    from oracle import dstt_oracle as O
    from paper_2509_10466_b200.weights import seed_parameters
    w = O.Params(cfg, seed_parameters(cfg, 0))
    steps = min(args.steps, 60 if cfg.width <= 512 else 4)
    warm = min(args.warmup, 1)
    zero = np.zeros((cfg.tokens, cfg.channels), np.float32)
    slots = (zero, zero)
    def one(i):
        if args.config == "C3":                     # stream 0, memory carried
            from paper_2509_10466_b200 import synth
            img, m = synth.C3Stream(0, cfg.width).frame(i)
            return img[None], m[None]
        return make_pool(args.config, 1, 0, cfg.width) if args.config != "C2" else _c2(i)
    frames = [one(i) for i in range(min(steps + warm, 8))]
    times = []
    for k in range(warm + steps):
        img, m = frames[k % len(frames)]
        t0 = time.perf_counter()
        res = O.inpaint_path(cfg, w, img, m, slots)
        dt = time.perf_counter() - t0
        if carried:
            slots = (slots[1], res["slot"][0])
        if k >= warm:
            times.append(dt)
    total = sum(times)
    value = steps / total
    line = {"metric": "inpainted frames/sec at 512x512 (p50 per-frame latency alongside)"
            if cfg.width == 512 else f"inpainted frames/sec at {cfg.width}x{cfg.width}",
            "impl": "reference", "value": value, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": 1e3 * total / steps,
            "p50_ms": 1e3 * statistics.median(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "global_batch": 1, "image": cfg.width,
                       "parallelism": "cpu"},
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores(),
                             "kind": "port", "sample": f"{steps} frames of {args.config}, "
                             f"numpy oracle (BLAS threads = host cores), {cpu_model()}"},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if steps != args.steps:
        line["note"] = f"capped at {steps} steps to bound CPU time (requested {args.steps})"
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2509_10466_b200 import DsttEngine, _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def allmax(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    cfg, B, carried, desc = workload(args.config, world)
    T, C, H, W = cfg.tokens, cfg.channels, cfg.height, cfg.width
    P = max(1, args.pool)
    if P % 3 == 0:                          # (k % P, k % 3) must cover every graph key
        P += 1
    t0 = time.perf_counter()
    imgs, masks = make_pool(args.config, P * B, rank, W, world)
    log(f"[bench] rank {rank}: pool of {P * B} frames in {time.perf_counter() - t0:.1f}s")
    eng = DsttEngine(cfg, seed=0, device=local)
    d_img = torch.from_numpy(imgs).to(dev).reshape(P, B, 3, H, W)
    d_msk = torch.from_numpy(masks.astype(np.uint8)).to(dev).reshape(P, B, H, W)
    ring = [torch.zeros((B, T, C), dtype=torch.float32, device=dev) for _ in range(3)]
    zero = torch.zeros((B, T, C), dtype=torch.float32, device=dev)
    out = torch.empty((B, 3, H, W), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def slots_for(k):
        """Memory FIFO over a 3-buffer ring: step k reads (k-2, k-1), writes k."""
        if not carried:
            return zero, zero, ring[k % 3]
        s0 = zero if k < 2 else ring[(k - 2) % 3]
        s1 = zero if k < 1 else ring[(k - 1) % 3]
        return s0, s1, ring[k % 3]

    def launch(k):
        s0, s1, ns = slots_for(k)
        eng.run(d_img[k % P], d_msk[k % P], (s0, s1), out={"out": out, "slot": ns},
                sync=False)

    # CUDA graphs of the whole path, one per (frame, ring state); memory is warm after
    # two steps, so graph keys are (k % P, k % 3) for k >= 2.
    stream = torch.cuda.Stream(dev)
    graphs = {}
    with torch.cuda.stream(stream):
        for k in range(3):
            launch(k)                      # allocate workspace, set kernel attributes
        torch.cuda.synchronize(dev)
        n_keys = P * 3 if carried else P
        for key in range(n_keys):
            k = key + 3 * P if carried else key
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                launch(k)
            graphs[(k % P, k % 3) if carried else k % P] = g

    def graph_for(k):
        k2 = k + 3 * P
        return graphs[(k2 % P, k2 % 3) if carried else k2 % P]

    kernels = eng.kernels_per_forward()
    with torch.cuda.stream(stream):
        for k in range(args.warmup):
            graph_for(k).replay()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        barrier()
        clocks = Clocks(local)
        w0 = time.perf_counter()
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            graph_for(args.warmup + k).replay()
            ev[k][1].record(stream)
        barrier()
        wall = time.perf_counter() - w0
        clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = allmax(sum(step_ms))
    value = world * args.steps * B / (total_ms / 1e3)
    p50 = statistics.median(step_ms)
    p99 = float(np.percentile(step_ms, 99))

    # live per-stage timing (un-graphed profiled pass over the same frames)
    lib = _lib.load()
    lib.dr_profile(eng.handle, 1)
    n_prof = min(args.steps, 50)
    acc = {}
    import ctypes
    msb = (ctypes.c_float * 64)()
    kinds = (ctypes.c_int32 * 64)()
    with torch.cuda.stream(stream):
        for k in range(n_prof):
            flush.zero_()
            launch(args.warmup + k + 3 * P)
            torch.cuda.synchronize(dev)
            n = lib.dr_profile_read(eng.handle, msb, kinds, 64)
            for i in range(max(n, 0)):
                name = _lib.STAGE_NAMES.get(kinds[i], str(kinds[i]))
                acc.setdefault(name, []).append(msb[i])
    lib.dr_profile(eng.handle, 0)
    flops = stage_flops(cfg)
    stages = {}
    prof_step = sum(sum(v) for v in acc.values()) / max(n_prof, 1)
    for name, v in acc.items():
        per_step = sum(v) / n_prof
        launches = len(v) / n_prof
        mean = sum(v) / len(v)
        stages[name] = {"ms_per_step": round(per_step, 5), "launches_per_step": launches,
                        "share": round(per_step / prof_step, 4) if prof_step else None,
                        "tflops": round(flops.get(name, 0) * B / (mean * 1e-3) / 1e12, 2)}
    dom = max(stages, key=lambda s: stages[s]["ms_per_step"]) if stages else None
    pk, pk_src = peaks()
    roof = None
    if dom:
        mean_ms = sum(acc[dom]) / len(acc[dom])
        if flops.get(dom, 0) > 0:
            ach = flops[dom] * B / (mean_ms * 1e-3) / 1e12
            roof = {"bound": "tensor", "kernel": dom, "achieved": round(ach, 2),
                    "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                    "frac": round(ach / pk["bf16_tflops"], 4),
                    "traffic": traffic(dom, B if args.config == "C2" else -1),
                    "peak_source": f"{pk_src} dense bf16 burst (MEASURED_PEAKS.json)",
                    "mean_launch_ms": round(mean_ms, 5)}
            if dom.startswith("attn_"):
                # head_dim 16: the binding unit is MUFU ex2 (16/clk/SM measured,
                # profiles/r01/pipe_microbench_b200.txt), not the tensor pipe
                exps = stage_exps(cfg)[dom] * B
                clk_hz = 1e6 * (clk["sm_mhz"] if clk and clk.get("sm_mhz") else pk.get("sm_max_mhz", 1965.0))
                mufu_peak = 16 * 148 * clk_hz
                roof["mufu"] = {"exps_per_launch": exps, "achieved_gexp_s": round(exps / (mean_ms * 1e-3) / 1e9, 1),
                                "peak_gexp_s": round(mufu_peak / 1e9, 1),
                                "frac": round(exps / (mean_ms * 1e-3) / mufu_peak, 4),
                                "note": "exponentials executed on MUFU + FMA-polynomial pipes"}
    path_tflops = frame_flops_reference(cfg) * B * args.steps / (sum(step_ms) * 1e-3) / 1e12

    # e2e through the reference-facing C-ABI call with host buffers (u8 API)
    e2e = None
    if B == 1:
        host_rgb = [np.ascontiguousarray((np.clip(np.rint(im.transpose(1, 2, 0) * 255), 0, 255))
                                         .astype(np.uint8)) for im in imgs]
        host_m = [np.ascontiguousarray(m.astype(np.uint8)) for m in masks]
        for i in range(P):
            host_rgb[i][host_m[i].astype(bool)] = 0           # reference API: redacted input
        eng.reset_host_memory()
        for k in range(min(args.warmup, 10)):
            eng.inpaint_host(host_rgb[k % P], host_m[k % P])
        barrier()
        d2h = 0
        host_ms = []
        e0 = time.perf_counter()
        for k in range(args.steps):
            t_k = time.perf_counter()
            eng.inpaint_host(host_rgb[k % P], host_m[k % P])
            host_ms.append(1e3 * (time.perf_counter() - t_k))
            d2h += lib.dr_host_d2h_bytes(eng.handle)
        e_s = allmax(time.perf_counter() - e0)
        e2e = {"value": world * args.steps / e_s, "unit": "frames/s",
               "h2d_bytes_per_step": H * W * 3 + H * W,
               "d2h_bytes_per_step": round(d2h / args.steps),
               "p50_ms_host": round(statistics.median(host_ms), 4),
               "p99_ms_host": round(float(np.percentile(host_ms, 99)), 4),
               "api": "dr_inpaint_u8_host (u8 HWC frame + mask in, u8 composite out, "
                      "engine-held memory; only the per-row spans within r+R of the mask are read back, packed)"}
    barrier()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, n, el = cpu_oracle_rate(args.config, args.cpu_seconds)
        cpu = {"value": rate * B if args.config != "C5" else rate, "unit": "frames/s",
               "cores": cores(), "kind": "port",
               "sample": f"{n} frames of {args.config} in {el:.1f}s, numpy oracle port of the "
                         f"reference path (BLAS threads = host cores), {cpu_model()}"}
    if rank == 0:
        line = {
            "metric": "inpainted frames/sec at 512x512 (p50 per-frame latency alongside)"
            if W == 512 else f"inpainted frames/sec at {W}x{W}",
            "value": round(value, 2), "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 5),
            "p50_ms": round(p50, 5), "p99_ms": round(p99, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f16", "data": "synthetic",
            "config": {"workload": desc, "global_batch": B * world, "image": W,
                       "parallelism": f"replicas x{world}" if world > 1 else "single",
                       "l2": "flushed between steps (256 MiB write), outside the step events",
                       "timing": "CUDA events around each step (CUDA-graph replay of the "
                                 "whole path); max over ranks", "pool_frames": P * B,
                       "bracket_wall_s": round(wall, 4)},
            "gpu_launches": kernels * args.steps,
            "path_tflops_dense": round(path_tflops, 2),
            "roofline": roof, "stages": stages,
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
