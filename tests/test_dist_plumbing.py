"""Multi-process plumbing of bench.py's N > 1 path on CPU (gloo, world size 2):
the ncclUniqueId broadcast from rank 0 and the max/sum-over-ranks timing
reductions. The GPU side of the partitioned solve is covered by
tests/test_gpu_dist.py (ranks emulated in one process)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    uid = bench.share_nccl_id(world, rank, lambda: bytes(range(128)))
    mx = bench.max_over_ranks(world, 10.0 + rank)
    sm = bench.sum_over_ranks(world, 1.5 * (rank + 1))
    bench.barrier(world)
    q.put((rank, uid == bytes(range(128)), mx, sm))
    dist.destroy_process_group()


def test_bench_distributed_plumbing_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, id_ok, mx, sm in out:
        assert id_ok
        assert mx == 11.0
        assert sm == 4.5
