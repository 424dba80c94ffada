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


def _tp_worker(rank, world, port, q):
    """Head-sharded decomposition on CPU (gloo): the shard plan the device model uses,
    row-parallel partial sums all-reduced, vocab shards gathered -> the unsharded result."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2311_04934_b200 as pcb
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nid = pcb.share_nccl_id(dist, make=lambda: bytes(range(128)))
    cfg = dict(n_heads=8, head_dim=16, vocab_size=96)
    d, V, n = 128, 96, 5
    plan = pcb.tp_shard_plan(cfg, world)[rank]
    rng = np.random.default_rng(0)  # same full tensors on every rank
    attn, x = rng.standard_normal((n, d)), rng.standard_normal((n, d))
    wo, w1, w2, un = (rng.standard_normal(s) for s in ((d, d), (4 * d, d), (d, 4 * d), (V, d)))
    gelu = lambda v: 0.5 * v * (1 + np.tanh(0.7978845608028654 * (v + 0.044715 * v ** 3)))  # noqa: E731
    a0, a1 = plan["wo_cols"]
    part_o = torch.tensor(attn[:, a0:a1] @ wo[:, a0:a1].T)
    r0, r1 = plan["w1_rows"]
    c0, c1 = plan["w2_cols"]
    part_m = torch.tensor(gelu(x @ w1[r0:r1].T) @ w2[:, c0:c1].T)
    dist.all_reduce(part_o)
    dist.all_reduce(part_m)
    u0, u1 = plan["unembed_rows"]
    shards = [torch.zeros(n, u1 - u0, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(shards, torch.tensor(x @ un[u0:u1].T))
    logits = torch.cat(shards, 1).numpy()
    ok = (np.allclose(part_o.numpy(), attn @ wo.T) and np.allclose(part_m.numpy(), gelu(x @ w1.T) @ w2.T)
          and np.allclose(logits, x @ un.T) and nid == bytes(range(128)))
    dist.destroy_process_group()
    q.put((rank, ok, plan["heads"]))


def test_tp_decomposition_gloo_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_tp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=180) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(o[1] for o in out)
    assert [o[2] for o in out] == [(0, 4), (4, 8)]


def test_bench_gpus2_relaunches_two_ranks_dry_run():
    """`bench.py --gpus 2` without torchrun re-launches itself with one process per rank; in the
    gloo dry run rank 0 prints exactly one JSON line that reports both ranks."""
    import json
    import subprocess

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                          "--steps", "4", "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["dry_run"] and line["steps"] == 4
    assert line["c4_requests_rank0"] == 256  # config 4 scales with the ranks: 256 requests per GPU
