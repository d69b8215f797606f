"""The N>1 path of bench.py on CPU: two gloo ranks shard the C4 pairs without
overlap and agree on the max-over-ranks time (the driver launches the GPU
version with torchrun, one rank per B200)."""

import os
import socket
import sys
from pathlib import Path

import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seeds = bench.rank_seeds(rank, pairs_per_step=16)
    t = bench.max_over_ranks(10.0 + rank, world)
    q.put((rank, seeds, t))
    dist.destroy_process_group()


def test_two_rank_sharding_and_max_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, (s, t)) for r, s, t in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s0, s1 = out[0][0], out[1][0]
    assert len(s0) == len(s1) == 16 * 2 and not set(s0) & set(s1)
    assert out[0][1] == out[1][1] == 11.0
