"""The N>1 path on CPU: world_size-2 gloo processes exercise the replica layout (disjoint
frame seeds / stream ownership, max-over-ranks timing, final gather) that bench.py uses
with NCCL on GPUs.  No data-path collective exists."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world_size, port, q):
    sys.path.insert(0, str(REPO))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world_size), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    from paper_2509_10466_b200 import replicas, synth
    r, ws, _ = replicas.world()
    seeds = replicas.frame_seeds(r, 3)
    streams = replicas.rank_streams(r, ws, 8)
    # each rank generates its own frames; no activation crosses ranks
    imgs = np.stack([synth.c2_frame(s, 64)[0] for s in seeds])
    t_local = 1.5 + r                              # per-rank "elapsed"
    t_max = replicas.allreduce_max(t_local)
    checksum = torch.tensor([float(imgs.sum())], dtype=torch.float64)
    gathered = replicas.gather_to_rank0(checksum)
    q.put((r, seeds, streams, t_max, None if gathered is None else [float(g) for g in gathered],
           float(imgs.sum())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(2):
        r, seeds, streams, t_max, gathered, local = q.get(timeout=240)
        results[r] = (seeds, streams, t_max, gathered, local)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s0, s1 = results[0][0], results[1][0]
    assert not set(s0) & set(s1)                                   # disjoint frames
    assert sorted(results[0][1] + results[1][1]) == list(range(8))  # every stream owned once
    assert results[0][1] == [0, 2, 4, 6]
    assert results[0][2] == results[1][2] == 2.5                   # max over ranks
    assert results[1][3] is None
    assert np.allclose(results[0][3], [results[0][4], results[1][4]])   # gather order = rank


def _bench_dry(*extra):
    import json
    import subprocess
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--dry-run",
                        "--steps", "2", "--warmup", "0", *extra],
                       capture_output=True, text=True, timeout=300, cwd=str(REPO))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_self_launches_two_ranks_c5_gloo():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks; C5 weak
    scaling shards 64 frames per rank (global batch 128), disjoint seeds, final gather of
    every rank's results to rank 0 in rank order."""
    d = _bench_dry("--config", "C5")
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 128
    assert d["ranks_gathered"] == [0, 1]
    assert d["frames_gathered"] == 2 * 64 * 2
    seeds = [s for s, _ in d["ids"]]
    assert len(set(seeds)) == len(seeds)
    assert seeds[:3] == [0, 1, 2] and seeds[128:131] == [100003, 100004, 100005]


def test_bench_self_launches_two_ranks_c3_streams_gloo():
    """C3 at 2 GPUs: streams round-robin over ranks (4 per rank, batched)."""
    d = _bench_dry("--config", "C3")
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 8
    owned0 = {s for s, _ in d["ids"][:8]}
    owned1 = {s for s, _ in d["ids"][8:]}
    assert owned0 == {0, 2, 4, 6} and owned1 == {1, 3, 5, 7}
