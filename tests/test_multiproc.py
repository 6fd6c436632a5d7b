"""CPU, world_size 2 over gloo: the replica harness of bench.py (barrier +
max-over-ranks timing; replicas only — the path has no data-path collective,
SURVEY.md §8(e)) and the reference arm's rank-0-only rule."""
import os
import socket
import sys
from pathlib import Path

import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import bench

    class A:
        impl = "reference"

    world_, rank_, local, pg = bench.dist_setup(A())
    assert (world_, rank_) == (world, rank)
    bench.barrier(pg, local)
    # each replica "measured" a different time; the job time is the max
    t = bench.allmax(pg, 10.0 + 5.0 * rank, local)
    q.put((rank, t))
    dist.destroy_process_group()


def test_replica_timing_is_max_over_ranks():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = dict(q.get() for _ in range(2))
    assert got == {0: 15.0, 1: 15.0}
