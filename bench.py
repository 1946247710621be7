#!/usr/bin/env python
"""Benchmark of the B200 masked-inpainting hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2|C1|C3|C4|C5] [--frames P] [--dry-run]

Default workload = BASELINE configs[1] (C2): batch-1 real-time path at 512x512, the
reference network (patch 8, C 64, 4 heads, S,T,S,T, temporal_groups 4) with seeded
random-init weights (seed 0), dilation r=5, feather sigma=3, memory carried across
frames, seeded synthetic frames (blurred-uniform image + ellipse/brush mask).  One step =
one frame (one batch for C3 / C5) through mask stage -> forward -> composite.

value     frames/s over all ranks, device time: CUDA events around every step (a CUDA
          graph replay of the whole path reading a static input buffer; the step's frame
          is copied in from the HBM-resident pool before the L2 flush, outside the events),
          L2 flushed (256 MiB write) between steps; p50/p99 per-frame latency alongside.
          The job total adds one final gather of the last step's composites to rank 0
          (NCCL gather; nothing at N=1) -- the only collective.
parity    the last timed step re-run eagerly on a second engine (fresh slot K/V
          projections): its composite and new slot must equal the graph replay bit for
          bit; one frame of it is checked against the CPU oracle (2e-2 max-abs, 40 dB).
e2e       frames/s through the reference-facing API with HOST buffers: the C-ABI host call
          (dr_inpaint_u8_host) and the drop-in `DsttEngine.inpaint(rgb, mask, memory)`
          (batch 1), or `DsttEngine.run` on pinned u8 frames (batches).
roofline  dominant kernel from per-stage CUDA events recorded INSIDE a CUDA graph of the
          same path (a second engine with event nodes between the launches).
cpu_baseline  the reference's own CPU implementation (baseline/ref_path.py: unmodified
          `dimreal` DsttModel + scipy masks) on this host, rank 0, bounded sample.

--impl reference: that reference CPU path alone on the same config, rank 0 only.
--gpus N > 1 without torchrun: re-launches itself under torch.distributed.run (one process
per GPU, NCCL); each rank owns whole frames / streams (weak scaling), barrier +
max-over-ranks timing.  --dry-run: the multi-rank plumbing on CPU (gloo) without kernels.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    p.add_argument("--frames", type=int, default=8,
                   help="distinct seeded frames (batches) per rank, cycled by the steps")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--dry-run", action="store_true",
                   help="multi-rank launch / sharding / gather on CPU (gloo), no kernels")
    return p.parse_args(argv)


# ---------------------------------------------------------------------------- launcher
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: re-run this command under torch.distributed.run with
    N processes on this node (rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    log("[bench] launching", args.gpus, "ranks:", " ".join(cmd[2:6]))
    return subprocess.run(cmd).returncode


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


def metric_name(size):
    return ("inpainted frames/sec at 512x512 (p50 per-frame latency alongside)" if size == 512
            else f"inpainted frames/sec at {size}x{size}")


def config_dict(name, world, batch, size):
    """The `config` object, identical for both arms of the same workload."""
    _, _, _, desc = workload(name, world)
    return {"workload": desc, "global_batch": batch * world, "image": size,
            "parallelism": f"replicas x{world} (frames/streams sharded by rank)" if world > 1
            else "single GPU",
            "l2": "inputs staged from an HBM pool, L2 flushed (256 MiB write) between steps"}


def stage_flops(cfg, kv_bands=3):
    """Dense algorithmic FLOPs per frame of each kernel class (per launch).  kv_bands: key
    bands a temporal query attends explicitly -- 3 with warm memory, 1 when both slots are
    the zero slot (their keys are one constant, dr_b200.h)."""
    T, C, H, W = cfg.tokens, cfg.channels, cfg.height, cfg.width
    g = cfg.temporal_groups
    tg = T // g
    dh = C // cfg.heads
    qkv = 2 * T * C * 3 * C
    return {
        "embed_qkv": 2 * T * (4 * cfg.patch ** 2) * C + qkv,
        "slot_kv": 2 * T * C * 2 * C,
        "attn_spatial": 2 * 2 * cfg.heads * T * T * dh,
        "attn_temporal": 2 * 2 * cfg.heads * g * tg * (kv_bands * tg) * dh,
        "mlp_qkv": 2 * T * (C * C + C * 2 * C + 2 * C * C) + qkv,
        "vec2patch": 2 * T * C * C * cfg.kernel ** 2,
        "decode0": 2 * H * W * C * C * 9,
        "decode2_composite": 2 * H * W * C * 3 * 9,
        "mask_stage": 0,
    }


def stage_bytes(cfg):
    """Algorithmic HBM bytes per frame of the HBM-class stages (device path: f32 rgb in).
    Mask stage: m0 u8 + rgb f32 in; alpha f32, token validity u8 and the packed fp16
    network input (4 channels per pixel) out.  Batch-1 decoder tail (decode.2 taps +
    composite): rgb f32 and alpha in, composite f32 out (its fp16 tap planes, an artefact of
    the unfused decomposition, are not counted)."""
    T, H, W = cfg.tokens, cfg.height, cfg.width
    return {"mask_stage": H * W * (1 + 12 + 4 + 8) + T,
            "decode2_composite": H * W * (12 + 4 + 12)}


def stage_exps(cfg, kv_bands=3):
    """Softmax exponentials per frame per attention launch (keys attended explicitly)."""
    T, g = cfg.tokens, cfg.temporal_groups
    tg = T // g
    return {"attn_spatial": cfg.heads * T * T,
            "attn_temporal": cfg.heads * g * tg * kv_bands * tg}


def frame_flops_reference(cfg, kv_bands=3):
    """Reference FlopCounterMode count per frame: the forward's dense
    contractions; attention counts QK^T and PV, linear layers once.  kv_bands=1: what runs
    with cold memory here (the zero slots' keys are one constant: no slot K/V projection,
    one key band per temporal query)."""
    f = stage_flops(cfg, kv_bands)
    T, C = cfg.tokens, cfg.channels
    n_s = sum(b == "S" for b in cfg.blocks)
    n_t = len(cfg.blocks) - n_s
    per_block_lin = 2 * T * (4 * C * C + 4 * C * C)     # q,k,v,out + ffn (64x128 x2)
    t_extra = 2 * 2 * T * 2 * C * C if kv_bands == 3 else 0   # k,v over both slots
    return (2 * T * 4 * cfg.patch ** 2 * C + len(cfg.blocks) * per_block_lin
            + n_s * f["attn_spatial"] + n_t * (f["attn_temporal"] + t_extra)
            + f["vec2patch"] + f["decode0"] + f["decode2_composite"])


def _gen(job):
    name, key, size = job
    from paper_2509_10466_b200 import synth
    if name == "C3":
        stream, t = key
        return synth.C3Stream(stream, size).frame(t)
    return {"C1": synth.c1_frame, "C2": synth.c2_frame, "C4": synth.c4_frame,
            "C5": synth.c5_frame}[name](key, size)


def make_pool(name, n, rank, size, world=1, procs=None):
    """n seeded frames of this rank (C3: n = frames x streams of this rank, time-major),
    generated in a process pool (numpy, ~0.2 s per 512^2 frame)."""
    if name == "C3":
        streams = [s for s in range(C3_STREAMS) if s % world == rank]
        keys = [(st, t) for t in range(n // len(streams)) for st in streams]
    else:
        keys = [rank * 100003 + i for i in range(n)]
    jobs = [(name, k, size) for k in keys]
    # (the ranks of one node generate their pools at the same time: share the host cores)
    procs = procs or min(len(jobs), max(1, ((os.cpu_count() or 2) - 1) // max(1, world)), 32)
    if procs > 1 and len(jobs) > 2:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_gen, jobs, chunksize=max(1, len(jobs) // (4 * procs)))
    else:
        res = [_gen(j) for j in jobs]
    return np.stack([r[0] for r in res]), np.stack([r[1] for r in res])


def traffic(stage, batch):
    """DRAM bytes per launch of `stage` from the committed ncu capture (batch-1 C2 frames,
    scripts/ncu_traffic.py), or None when there is no capture for this workload."""
    for rnd in ("r02", "r01"):
        p = REPO / "profiles" / rnd / "ncu_traffic.json"
        if batch == 1 and p.exists():
            st = json.loads(p.read_text())["stages"].get(stage)
            return None if st is None else round(st["dram_bytes_per_launch"])
    return None


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


def cpu_frames(name, n):
    """A small sample of the workload's frames for the CPU path (one stream for C3)."""
    if name == "C3":
        from paper_2509_10466_b200 import synth
        st = synth.C3Stream(0)
        return [st.frame(t) for t in range(n)]
    imgs, masks = make_pool(name, n, 0, workload(name)[0].width)
    return list(zip(imgs, masks))


class CpuPath:
    """The reference's own CPU implementation (kind "reference"); the numpy oracle port
    only if the reference install is missing (kind "port")."""

    def __init__(self, name):
        cfg, _, carried, _ = workload(name)
        self.carried = carried
        from baseline import ref_path
        why = ref_path.available()
        if why is None:
            self.kind = "reference"
            self.path = ref_path.ReferencePath(cfg.width, cfg.mask_dilate,
                                               cfg.mask_feather_sigma, threads=cores())
            self.threads = self.path.threads
            self.what = ("unmodified dimreal DsttModel (baseline/_ref, torch CPU, "
                         f"{self.threads} threads) + scipy binary_dilation(_CROSS) / "
                         "gaussian_filter + fp32 composite")
            if cfg.mask_aware_attention:
                self.what += " (plain attention: the reference has no mask-aware mode)"
        else:
            from oracle import dstt_oracle as O
            from paper_2509_10466_b200.weights import seed_parameters
            self.kind = "port"
            self.why = why
            self.O, self.cfg = O, cfg
            self.w = O.Params(cfg, seed_parameters(cfg, 0))
            z = np.zeros((cfg.tokens, cfg.channels), np.float32)
            self.slots = (z, z)
            self.threads = cores()
            self.what = f"numpy oracle port (reference install missing: {why})"

    def step(self, img, m0):
        if self.kind == "reference":
            return self.path.step(img, m0, self.carried)
        res = self.O.inpaint_path(self.cfg, self.w, img[None], m0[None], self.slots)
        if self.carried:
            self.slots = (self.slots[1], res["slot"][0])
        return res["out"][0]


def cpu_rate(name, seconds, max_frames=64):
    """CPU path frames/s over a bounded sample (about `seconds` of work after one warm-up
    frame)."""
    path = CpuPath(name)
    frames = cpu_frames(name, 4)
    path.step(*frames[0])
    n, t0 = 0, time.perf_counter()
    while True:
        path.step(*frames[n % len(frames)])
        n += 1
        el = time.perf_counter() - t0
        if (el >= seconds and n >= 2) or n >= max_frames:
            break
    return n / el, n, el, path


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    cfg, batch, carried, desc = workload(args.config, world)
    path = CpuPath(args.config)
    per_frame_s = {256: 0.08, 512: 0.6, 1024: 8.0}[cfg.width]
    budget = 150.0                                    # seconds of timed CPU work at most
    steps = max(2, min(args.steps, int(budget / per_frame_s) - args.warmup))
    frames = cpu_frames(args.config, min(8, steps + args.warmup))
    times = []
    for k in range(args.warmup + steps):
        img, m0 = frames[k % len(frames)]
        t0 = time.perf_counter()
        path.step(img, m0)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    total = sum(times)
    value = steps / total
    line = {"metric": metric_name(cfg.width), "impl": "reference", "value": value,
            "unit": "frames/s", "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / steps, "p50_ms": 1e3 * statistics.median(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": config_dict(args.config, world, batch, cfg.width),
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": path.threads,
                             "kind": path.kind,
                             "sample": f"{steps} frames of {args.config} (one stream / one "
                                       f"frame per step, memory carried={carried}), "
                                       f"{path.what}, {cpu_model()}"},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if steps != args.steps:
        line["note"] = f"capped at {steps} steps to bound CPU time (requested {args.steps})"
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- dry run
def run_dry(args):
    """The N-rank plumbing without GPU kernels: gloo process group, per-rank shard of the
    workload (frame seeds / streams), a stand-in step per shard, max-over-ranks timing and
    the final gather to rank 0 -- what run_ours does around the kernels."""
    import torch
    import torch.distributed as dist

    from paper_2509_10466_b200 import replicas
    rank, world, _ = replicas.world()
    if world > 1:
        dist.init_process_group("gloo")
    cfg, B, carried, desc = workload(args.config, world)
    if args.config == "C3":
        owned = replicas.rank_streams(rank, world, C3_STREAMS)
        ids = [[s, t] for t in range(args.steps) for s in owned]
    else:
        ids = [[s, 0] for s in replicas.frame_seeds(rank, B * args.steps)]
    t0 = time.perf_counter()
    # stand-in result per frame: (rank, seed / stream, step)
    out = torch.tensor([[rank, s, t] for s, t in ids], dtype=torch.int64)
    el = replicas.allreduce_max(time.perf_counter() - t0)
    got = replicas.gather_to_rank0(out)
    if rank == 0:
        allf = torch.cat(got)
        print(json.dumps({"dry_run": True, "metric": metric_name(cfg.width), "value": None,
                          "n_gpus": world, "steps": args.steps,
                          "config": config_dict(args.config, world, B, cfg.width),
                          "frames_gathered": int(allf.shape[0]),
                          "ranks_gathered": sorted({int(r) for r in allf[:, 0]}),
                          "ids": allf[:, 1:].tolist(), "max_rank_s": el}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2509_10466_b200 import BinaryMask, DsttEngine, _lib, replicas

    rank, world, local = replicas.world()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    cfg, B, carried, desc = workload(args.config, world)
    T, C, H, W = cfg.tokens, cfg.channels, cfg.height, cfg.width
    P = max(1, args.frames)
    t0 = time.perf_counter()
    imgs, masks = make_pool(args.config, P * B, rank, W, world)
    log(f"[bench] rank {rank}: pool of {P * B} frames in {time.perf_counter() - t0:.1f}s")
    eng = DsttEngine(cfg, seed=0, device=local)
    d_img = torch.from_numpy(imgs).to(dev).reshape(P, B, 3, H, W)
    d_msk = torch.from_numpy(masks.astype(np.uint8)).to(dev).reshape(P, B, H, W)
    x_img = torch.empty((B, 3, H, W), dtype=torch.float32, device=dev)   # graph inputs
    x_msk = torch.empty((B, H, W), dtype=torch.uint8, device=dev)
    ring = [torch.zeros((B, T, C), dtype=torch.float32, device=dev) for _ in range(3)]
    out = torch.empty((B, 3, H, W), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def slots_for(k, e=None):
        """Memory FIFO over a 3-buffer ring: step k reads (k-2, k-1), writes k.  Cold slots
        are engine e's zero slot (InpaintMemory.from_zero_slot, memory.py:32-34)."""
        zero = (e or eng).zero_memory().slots[0]     # [T][C], shared by every frame
        if not carried:
            return zero, zero, ring[0]
        s0 = zero if k < 2 else ring[(k - 2) % 3]
        s1 = zero if k < 1 else ring[(k - 1) % 3]
        return s0, s1, ring[k % 3]

    def stage(k):
        x_img.copy_(d_img[k % P])
        x_msk.copy_(d_msk[k % P])
    stage.inputs = (x_img, x_msk)

    def launch(e, k, o=None, ns=None, clone=False):
        s0, s1, w = slots_for(k, e)
        if clone:
            s0, s1 = s0.clone(), s1.clone()
        e.run(x_img, x_msk, (s0, s1), out={"out": out if o is None else o,
                                           "slot": w if ns is None else ns}, sync=False)

    # Whole-path CUDA graphs reading the static input buffers: one per ring state (the
    # slot pointers and the slot K/V cache decisions are baked in), captured in the cyclic
    # order they replay in; memory is warm after two steps.
    n_keys = 3 if carried else 1
    stream = torch.cuda.Stream(dev)

    def capture(e):
        gs = []
        with torch.cuda.stream(stream):
            for k in range(3):
                stage(k)
                launch(e, k)                 # allocate workspace, warm the cache
            torch.cuda.synchronize(dev)
            for k in range(3, 3 + n_keys):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    launch(e, k)
                gs.append(g)
        return gs

    graphs = capture(eng)
    kernels = eng.kernels_per_forward()
    K, Wm = args.steps, args.warmup
    with torch.cuda.stream(stream):
        for k in range(Wm):
            stage(k)
            graphs[k % n_keys].replay()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
        barrier()
        clocks = Clocks(local)
        w0 = time.perf_counter()
        for i in range(K):
            k = Wm + i
            stage(k)
            flush.zero_()
            ev[i][0].record(stream)
            graphs[k % n_keys].replay()
            ev[i][1].record(stream)
        # the only collective: one final gather of the last step's composites to rank 0
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        gathered = replicas.gather_to_rank0(out) if world > 1 else [out]
        g1.record(stream)
        barrier()
        wall = time.perf_counter() - w0
        clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    gather_ms = g0.elapsed_time(g1) if world > 1 else 0.0
    total_ms = replicas.allreduce_max(sum(step_ms) + gather_ms, dev)
    value = world * K * B / (total_ms / 1e3)
    p50 = statistics.median(step_ms)
    p99 = float(np.percentile(step_ms, 99))
    k_last = Wm + K - 1
    # s0, s1 (None = the zero slot), new slot, out
    z = eng.zero_memory().slots[0]
    last = [None if t is z else t.clone() for t in slots_for(k_last)] + [out.clone()]

    # ---- per-stage times inside a CUDA graph (second engine, event nodes per stage)
    lib = _lib.load()
    eng_p = DsttEngine(cfg, seed=0, device=local)
    lib.dr_profile(eng_p.handle, 1)
    pgraphs = capture(eng_p)
    n_prof = min(K, 30)
    acc = {}
    msb = (ctypes.c_float * 64)()
    kinds = (ctypes.c_int32 * 64)()
    prof_ms = []
    with torch.cuda.stream(stream):
        for i in range(n_prof):
            k = Wm + i
            stage(k)
            flush.zero_()
            pgraphs[k % n_keys].replay()
            torch.cuda.synchronize(dev)
            n = lib.dr_profile_read(eng_p.handle, msb, kinds, 64)
            prof_ms.append(sum(msb[j] for j in range(max(n, 0))))
            for j in range(max(n, 0)):
                name = _lib.STAGE_NAMES.get(kinds[j], str(kinds[j]))
                acc.setdefault(name, []).append(msb[j])
    lib.dr_profile(eng_p.handle, 0)
    kv_bands = 3 if carried else 1           # cold memory: both slots are the zero slot
    flops = stage_flops(cfg, kv_bands)
    stages = {}
    prof_step = statistics.mean(prof_ms) if prof_ms else 0.0
    for name, v in acc.items():
        per_step = sum(v) / n_prof
        mean = sum(v) / len(v)
        stages[name] = {"ms_per_step": round(per_step, 5), "launches_per_step": len(v) / n_prof,
                        "share": round(per_step / prof_step, 4) if prof_step else None,
                        "tflops": round(flops.get(name, 0) * B / (mean * 1e-3) / 1e12, 2)}
        nbytes = stage_bytes(cfg).get(name)
        if nbytes:                       # HBM-class stage: achieved GB/s vs the copy peak
            gbs = nbytes * B / (mean * 1e-3) / 1e9
            stages[name].update({"gbs": round(gbs, 1),
                                 "hbm_frac": round(gbs / peaks()[0]["hbm_gbs"], 4)})
    dom = max(stages, key=lambda s: stages[s]["ms_per_step"]) if stages else None
    pk, pk_src = peaks()
    roof = None
    if dom:
        mean_ms = sum(acc[dom]) / len(acc[dom])
        ach = flops.get(dom, 0) * B / (mean_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": dom, "achieved": round(ach, 2),
                "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": round(ach / pk["bf16_tflops"], 4),
                "traffic": traffic(dom, B if args.config == "C2" else -1),
                "peak_source": f"{pk_src} dense bf16 burst (MEASURED_PEAKS.json)",
                "mean_launch_ms": round(mean_ms, 5),
                "timing": "CUDA events recorded inside a graph of the same path (event "
                          "nodes between launches break PDL overlap at the stage borders)"}
        if dom.startswith("attn_"):
            # head_dim 16: the binding unit is MUFU ex2 (16/clk/SM measured,
            # profiles/r01/pipe_microbench_b200.txt), not the tensor pipe
            exps = stage_exps(cfg, kv_bands)[dom] * B
            clk_hz = 1e6 * (clk["sm_mhz"] if clk and clk.get("sm_mhz") else 1965.0)
            mufu_peak = 16 * 148 * clk_hz
            roof["mufu"] = {"exps_per_launch": exps,
                            "achieved_gexp_s": round(exps / (mean_ms * 1e-3) / 1e9, 1),
                            "peak_gexp_s": round(mufu_peak / 1e9, 1),
                            "frac": round(exps / (mean_ms * 1e-3) / mufu_peak, 4),
                            "note": "exponentials executed on MUFU + FMA-polynomial pipes"}
    path_tflops = frame_flops_reference(cfg) * B * K / (sum(step_ms) * 1e-3) / 1e12

    # ---- parity of the timed output: eager re-run of the last step on the second engine
    parity = None
    if not args.no_parity:
        parity = check_parity(eng_p, cfg, B, stage, k_last, last, imgs, masks, P, rank, dev,
                              stream)

    # ---- e2e through the reference-facing API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(args, eng, cfg, B, imgs, masks, P, world, dev, barrier, lib,
                          BinaryMask)
    barrier()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, n, el, path = cpu_rate(args.config, args.cpu_seconds)
        cpu = {"value": rate, "unit": "frames/s", "cores": path.threads, "kind": path.kind,
               "sample": f"{n} frames of {args.config} in {el:.1f}s (one frame per step, "
                         f"memory carried={carried}), {path.what}, {cpu_model()}"}
    if rank == 0:
        line = {
            "metric": metric_name(W),
            "value": round(value, 2), "unit": "frames/s", "n_gpus": world,
            "steps": K, "warmup": Wm, "ms_per_step": round(total_ms / K, 5),
            "p50_ms": round(p50, 5), "p99_ms": round(p99, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f16", "data": "synthetic",
            "config": config_dict(args.config, world, B, W),
            "timing": "CUDA events around each step (CUDA-graph replay of the whole path); "
                      "job total = max over ranks of (sum of steps + final gather)",
            "frames_distinct": P * B, "bracket_wall_s": round(wall, 4),
            "final_gather": {"ms": round(gather_ms, 4),
                             "bytes": int(out.numel() * out.element_size() * (world - 1)),
                             "how": "NCCL gather of the last step's composites to rank 0"
                             if world > 1 else "none (single rank)"},
            "gpu_launches": kernels * K,
            "path_tflops_dense": round(path_tflops, 2),
            "roofline": roof, "stages": stages,
            "profiled_graph_ms_per_step": round(prof_step, 5),
            "parity": parity,
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    del gathered
    if world > 1:
        dist.destroy_process_group()


def check_parity(eng2, cfg, B, stage, k_last, last, imgs, masks, P, rank, dev, stream):
    """Re-run the last timed step eagerly on a second engine with copies of its memory
    slots (fresh slot K/V projections, no graph; a zero slot stays that engine's zero
    slot): composite and new slot must be bit-equal to the graph replay.  Then frame 0 of
    that step against the CPU oracle (2e-2 max-abs, 40 dB) given the same memory."""
    import torch
    s0, s1, last_slot, last_out = last
    out2 = torch.empty_like(last_out)
    ns2 = torch.empty_like(last_slot)
    zero = eng2.zero_memory().slots[0]
    mem = tuple(zero if s is None else s.clone() for s in (s0, s1))
    with torch.cuda.stream(stream):
        stage(k_last)
        eng2.run(*_inputs_of(stage), mem, out={"out": out2, "slot": ns2}, sync=False)
    torch.cuda.synchronize(dev)
    bit_out = bool(torch.equal(out2, last_out))
    bit_slot = bool(torch.equal(ns2, last_slot))
    res = {"step": k_last, "graph_vs_eager_bitexact": bit_out and bit_slot, "frames": B}
    if rank == 0:
        from oracle import dstt_oracle as O
        from paper_2509_10466_b200.weights import seed_parameters
        sl = tuple((s if s.dim() == 2 else s[0]).cpu().numpy() for s in mem)
        i = (k_last % P) * B
        t0 = time.perf_counter()
        ref = O.inpaint_path(cfg, seed_parameters(cfg, 0), imgs[i:i + 1], masks[i:i + 1], sl)
        got = last_out[0:1].cpu().numpy().astype(np.float64)
        err = float(np.max(np.abs(got - ref["out"])))
        mse = float(np.mean((got - ref["out"]) ** 2))
        ps = float("inf") if mse == 0 else 10 * np.log10(1.0 / mse)
        res.update({"oracle_frame": int(i), "oracle_max_abs": round(err, 6),
                    "oracle_psnr_db": round(ps, 2), "oracle_s": round(time.perf_counter() - t0, 1),
                    "tolerance": "max-abs <= 2e-2, PSNR >= 40 dB (north_star)"})
        res["pass"] = bool(res["graph_vs_eager_bitexact"] and err <= 2e-2 and ps >= 40.0)
    return res


def measure_e2e(args, eng, cfg, B, imgs, masks, P, world, dev, barrier, lib, BinaryMask):
    """Same metric end to end through the public API with host buffers: every step copies
    that step's u8 frame + mask host->device and the u8 composite device->host."""
    import torch

    from paper_2509_10466_b200 import replicas
    H, W = cfg.height, cfg.width
    K = args.steps
    host_rgb = np.ascontiguousarray(np.clip(np.rint(imgs.transpose(0, 2, 3, 1) * 255), 0, 255)
                                    .astype(np.uint8))
    host_m = np.ascontiguousarray(masks.astype(np.uint8))
    host_rgb[masks] = 0                                   # reference API: redacted input
    res = {"unit": "frames/s", "h2d_bytes_per_step": B * (H * W * 3 + H * W)}
    if B == 1:
        # (1) the C-ABI host call, engine-held memory
        eng.reset_host_memory()
        for k in range(min(args.warmup, 10)):
            eng.inpaint_host(host_rgb[k % P], host_m[k % P])
        barrier()
        d2h, host_ms = 0, []
        e0 = time.perf_counter()
        for k in range(K):
            t_k = time.perf_counter()
            eng.inpaint_host(host_rgb[k % P], host_m[k % P])
            host_ms.append(1e3 * (time.perf_counter() - t_k))
            d2h += lib.dr_host_d2h_bytes(eng.handle)
        e_s = replicas.allreduce_max(time.perf_counter() - e0, dev)
        res.update({"value": world * K / e_s, "d2h_bytes_per_step": round(d2h / K),
                    "p50_ms_host": round(statistics.median(host_ms), 4),
                    "p99_ms_host": round(float(np.percentile(host_ms, 99)), 4),
                    "api": "dr_inpaint_u8_host (u8 HWC frame + mask in, u8 composite out, "
                           "engine-held memory; only the per-row spans within r+R of the "
                           "mask are read back, packed)"})
        # (2) the drop-in reference signature: inpaint(rgb, BinaryMask, memory)
        bm = [BinaryMask(masks[i]) for i in range(P)]
        mem = eng.zero_memory()
        for k in range(min(args.warmup, 10)):
            mem = eng.inpaint(host_rgb[k % P], bm[k % P], mem).memory
        barrier()
        host_ms = []
        e0 = time.perf_counter()
        for k in range(K):
            t_k = time.perf_counter()
            mem = eng.inpaint(host_rgb[k % P], bm[k % P], mem).memory
            host_ms.append(1e3 * (time.perf_counter() - t_k))
        e_s = replicas.allreduce_max(time.perf_counter() - e0, dev)
        res["dropin"] = {"value": world * K / e_s, "unit": "frames/s",
                         "p50_ms_host": round(statistics.median(host_ms), 4),
                         "api": "DsttEngine.inpaint(rgb u8 HWC, BinaryMask, InpaintMemory) "
                                "-> EngineResult (base.py:52-89 signature, what "
                                "LocalEngineClient.inpaint_frame calls)"}
        # (3) a video stream through BatchStreamer (batch 1, memory carried): frame k+1's
        # upload and frame k-1's download overlap frame k's forward (one frame of lookahead)
        e_s = _streamed(args, eng, 1, host_rgb, host_m, P, K, True, barrier, dev)
        res["streamed"] = {"value": world * K / e_s, "unit": "frames/s",
                           "d2h_bytes_per_step": H * W * 3, "api": STREAMED_API}
        return res
    # batches: BatchStreamer (DsttEngine.run per batch) on pinned u8 frames, u8 composite
    # back to pinned memory; the next batch's upload and the previous batch's download
    # overlap the current forward (copy streams), every copy inside the timed region
    e_s = _streamed(args, eng, B, host_rgb, host_m, P, K, workload_carried(args.config),
                    barrier, dev)
    res.update({"value": world * K * B / e_s, "d2h_bytes_per_step": B * H * W * 3,
                "api": STREAMED_API})
    return res


STREAMED_API = ("BatchStreamer.submit (DsttEngine.run per batch) on u8 (B,H,W,3) pinned host "
                "frames + masks, per-stream memory -> u8 composite in pinned host memory; "
                "upload of batch k+1 and download of batch k-1 overlap the forward of batch k "
                "(streaming.py); steps run back to back with no L2 flush between them, so "
                "this figure can exceed the L2-flushed device value")


def _streamed(args, eng, B, host_rgb, host_m, P, K, carried, barrier, dev):
    """K batches through BatchStreamer from pinned host memory; seconds (max over ranks).
    Carried memory: the streamer's own per-stream FIFO with graph replays in steady state
    (warm-up covers the graph captures)."""
    import torch

    from paper_2509_10466_b200 import replicas
    from paper_2509_10466_b200.streaming import BatchStreamer
    H, W = host_m.shape[1:3]
    pin_rgb = torch.from_numpy(host_rgb).reshape(P, B, H, W, 3).pin_memory()
    pin_m = torch.from_numpy(host_m).reshape(P, B, H, W).pin_memory()
    pin_out = [torch.empty((B, H, W, 3), dtype=torch.uint8).pin_memory() for _ in range(2)]
    bs = BatchStreamer(eng, B, carry_memory=carried)

    def one(k):
        bs.submit(pin_rgb[k % P], pin_m[k % P], pin_out[k & 1])
    for k in range(BatchStreamer.GRAPH_WARM + 6 if carried else min(args.warmup, 10)):
        one(k)
    bs.finish()
    barrier()
    e0 = time.perf_counter()
    for k in range(K):
        one(k)
    bs.finish()
    return replicas.allreduce_max(time.perf_counter() - e0, dev)


def _inputs_of(stage):
    return stage.inputs


def workload_carried(name):
    return name in ("C1", "C2", "C3", "C4")


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N ranks with "
                         "torchrun --nproc-per-node N (or without torchrun to self-launch)")
    if world > 1 and not args.dry_run:
        # NCCL communicator lines (nranks) on stderr, stdout stays one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.impl == "reference":
        run_reference(args)
    elif args.dry_run:
        run_dry(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
