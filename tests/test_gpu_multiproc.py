"""Multi-process paths on the device.

* Head-sharded serving with one PROCESS per rank over the peer-memory transport (CUDA IPC
  buffers + one-shot all-reduce / all-gather kernels): runs on ONE GPU with both ranks
  sharing it, so the multi-process plumbing (handle exchange through torch.distributed,
  lockstep store / serve calls, system-scope flags) is exercised on every GPU run.
* The same over NCCL, and the data-parallel bench with 2 ranks: need 2 GPUs (skipped on 1).
Every sharded result must agree across ranks and match the unsharded model
(bf16 rel <= 2e-2, same greedy tokens)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2311_04934_b200 as pcb
from tests.util import BF16_REL, rel, same_greedy_token

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = dict(n_layers=2, n_heads=4, head_dim=64, hidden=256, vocab_size=512, pos_encoding="rope", max_position=8192,
           bytes_per_element=2, seed=42)
SCHEMA = ('<schema name="mp"><module name="sys">You answer from the documents below. </module>'
          '<module name="doc">The Seine flows through Paris; the Thames through London; the Tiber '
          'through Rome.</module></schema>')
PROMPTS = ['<prompt schema="mp"><sys/><doc/>Which river runs through Rome?</prompt>',
           '<prompt schema="mp"><doc/>Name a city.</prompt>']


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, transport, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2311_04934_b200 as pcb
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = 0 if transport == "peer" else rank  # "peer": both ranks share GPU 0
        if transport in ("peer", "peer_gpus"):
            peer = pcb.peer_group(dist, device=dev, cap_floats=1 << 20)
            m = pcb.Model(CFG, dtype=pcb.BF16, peer=peer)
        else:
            nid = pcb.share_nccl_id(dist)
            m = pcb.Model(CFG, dtype=pcb.BF16, device=dev, tp_rank=rank, tp_size=world, nccl_id=nid)
        schema = pcb.Schema.parse(SCHEMA)
        store = pcb.ModuleStore(m)
        store.encode_schema(schema)
        out = []
        for p in PROMPTS:
            r = pcb.serve(store, schema, p, max_new_tokens=4)
            out.append((r.output_tokens, r.first_token_logits.tolist()))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, repr(e)))


def _run_ranks(world, transport):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank, args=(r, world, port, transport, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
    errs = [e for _, _, e in res if e]
    assert not errs, errs
    return [o for _, o, _ in res]


def _check_against_unsharded(outs):
    m = pcb.Model(CFG, dtype=pcb.BF16)
    schema = pcb.Schema.parse(SCHEMA)
    store = pcb.ModuleStore(m)
    store.encode_schema(schema)
    for i, p in enumerate(PROMPTS):
        want = pcb.serve(store, schema, p, max_new_tokens=4)
        for o in outs:  # every rank holds the full (gathered) logits and the same tokens
            assert o[i][0] == outs[0][i][0]
            assert np.array_equal(np.asarray(o[i][1]), np.asarray(outs[0][i][1]))
        got = np.asarray(outs[0][i][1], np.float32)
        assert rel(got, want.first_token_logits) <= BF16_REL
        assert same_greedy_token(got, want.first_token_logits, f"tp multiprocess prompt {i}")


def test_tp_two_processes_peer_memory_one_gpu():
    _check_against_unsharded(_run_ranks(2, "peer"))


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_tp_two_processes_nccl():
    _check_against_unsharded(_run_ranks(2, "nccl"))


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_tp_two_gpus_peer_memory():
    # one process per GPU, peer loads over NVLink
    _check_against_unsharded(_run_ranks(2, "peer_gpus"))


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_bench_two_ranks_data_parallel():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                          "--skip-cpu", "--skip-slow", "--skip-c3", "--skip-sweep", "--micro-batches", "32"],
                         capture_output=True, text=True, timeout=1200, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["batch"]["requests"] == 512


def test_bench_two_ranks_data_parallel_share_one_gpu():
    """Data-parallel bench path as two processes (replicas on GPU 0, gloo plumbing): per-rank
    request streams, every rank's model / store / micro-batches, barrier + max-over-ranks timing
    and rank 0's single JSON line.  Functional only -- the ranks time-slice one GPU."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--share-device", "--steps", "3",
                          "--warmup", "3", "--skip-cpu", "--skip-slow", "--skip-c3", "--skip-sweep",
                          "--micro-batches", "16"],
                         capture_output=True, text=True, timeout=1200, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["ranks_share_one_gpu"]
    assert line["config"]["parallelism"] == "dp2" and line["batch"]["requests"] == 512
