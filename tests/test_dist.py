"""N>1 plumbing of bench.py on CPU: world_size-2 gloo group, barrier, max-over-ranks timing and the
per-rank request stream (DP replicas, weak scaling: no collective on the data path)."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    D = bench.Dist(backend="gloo")
    D.barrier()
    m = D.max(10.0 + rank)          # per-rank region time -> job time is the max
    reqs = D.requests(6, 4)
    # whole-job value as bench.py computes it: world * steps / max(region)
    value = D.world * 6 / m
    D.barrier()
    D.close()
    q.put((rank, m, reqs, value))


def test_dist_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[1] for o in out] == [11.0, 11.0]            # max over ranks, seen by every rank
    assert out[0][2] == [0, 1, 2, 3, 0, 1]                 # rank 0: requests 0..5 of the stream
    assert out[1][2] == [2, 3, 0, 1, 2, 3]                 # rank 1: requests 6..11 of the stream
    assert out[0][3] == pytest.approx(2 * 6 / 11.0)


def test_dist_single_rank_is_local():
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        os.environ.pop(k, None)
    sys.path.insert(0, ROOT)
    import bench
    D = bench.Dist()
    assert (D.world, D.rank) == (1, 0)
    assert D.max(3.5) == 3.5
    assert D.requests(3, 4) == [0, 1, 2]
    D.close()
