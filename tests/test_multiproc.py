"""Multi-process host logic on CPU (gloo, world_size 2, 127.0.0.1).

* The tensor-parallel decomposition the GPU path uses (``parallel.tp_slices``,
  mirrored by nfb_create_tp / nfb_synth_block_weights): each rank computes the
  split-K partial of its heads / FFN rows / vocab rows with the float64
  oracle, a gloo all-reduce sums them, and the sum must equal the unsharded
  oracle block (and logits).
* The bench's collectives: max-over-ranks timing and the NCCL-unique-id
  broadcast.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import neox_oracle as O
from paper_2604_23553_b200 import ModelConfig
from paper_2604_23553_b200.parallel import broadcast_bytes, max_over_ranks, tp_slices

CFG = dict(hidden=64, n_heads=4, d_head=16, n_layers=1, d_mlp=128, rotary_pct=0.25, vocab=96)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_partial(x, p, kv, pos, s, sl):
    """This rank's share of the parallel-residual block output (nf/golden.py:210-228)."""
    n1 = O.ln_two_pass(x, p["ln1_gain"], p["ln1_bias"], s.ln_eps)
    r0, r1 = sl.qkv_rows
    y = (p["qkv_weight"][r0:r1] @ n1 + p["qkv_bias"][r0:r1]).reshape(-1, 3 * s.d_head)
    d = s.d_head
    q = O.rope(y[:, :d], pos, s.rotary_dims, s.theta_base)
    k = O.rope(y[:, d:2 * d], pos, s.rotary_dims, s.theta_base)
    v = y[:, 2 * d:]
    hs, he = sl.heads
    keys = np.concatenate([kv[0][hs:he], k[:, None]], 1)
    vals = np.concatenate([kv[1][hs:he], v[:, None]], 1)
    ctx = np.concatenate([O.attend(q[i], keys[i], vals[i], 1.0 / math.sqrt(d)) for i in range(he - hs)])
    c0, c1 = sl.out_cols
    out = p["out_weight"][:, c0:c1] @ ctx
    n2 = O.ln_two_pass(x, p["ln2_gain"], p["ln2_bias"], s.ln_eps)
    m0, m1 = sl.mlp_rows
    g = O.gelu(p["up_weight"][m0:m1] @ n2 + p["up_bias"][m0:m1])
    out = out + p["down_weight"][:, m0:m1] @ g
    if sl.root:
        out = out + x + p["out_bias"] + p["down_bias"]
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = ModelConfig(**CFG)
        s = O.Shape.of(cfg)
        p = O.synth_block(s, 11)
        head = O.synth_head(s, 12)
        rng = np.random.default_rng(3)
        pos = 9
        kv = (rng.standard_normal((s.n_heads, pos, s.d_head)) * 0.5,
              rng.standard_normal((s.n_heads, pos, s.d_head)) * 0.5)
        x = rng.standard_normal(s.hidden) * 0.5
        sl = tp_slices(cfg, rank, world)
        part = torch.from_numpy(_shard_partial(x, p, kv, pos, s, sl))
        dist.all_reduce(part)  # the per-layer NCCL all-reduce of the GPU path
        h = part.numpy()
        v0, v1 = sl.vocab_rows
        hn = O.ln_two_pass(h, head["lnf_gain"], head["lnf_bias"], s.ln_eps)
        logits = torch.from_numpy(head["unembed"][v0:v1] @ hn)
        gathered = [torch.empty_like(logits) for _ in range(world)]
        dist.all_gather(gathered, logits)
        t = max_over_ranks(0.5 + rank)
        uid = broadcast_bytes(bytes(range(128)) if rank == 0 else None, 128)
        q.put((rank, h, torch.cat(gathered).numpy(), t, uid))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_tensor_parallel_decomposition_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=100) for _ in range(world))
    for pr in procs:
        pr.join(30)
        assert pr.exitcode == 0
    cfg = ModelConfig(**CFG)
    s = O.Shape.of(cfg)
    p = O.synth_block(s, 11)
    head = O.synth_head(s, 12)
    rng = np.random.default_rng(3)
    pos = 9
    kv = O.KV.of(rng.standard_normal((s.n_heads, pos, s.d_head)) * 0.5,
                 rng.standard_normal((s.n_heads, pos, s.d_head)) * 0.5)
    x = rng.standard_normal(s.hidden) * 0.5
    want = O.block_step(x, p, kv, pos, s)
    want_logits = head["unembed"] @ O.ln_two_pass(want, head["lnf_gain"], head["lnf_bias"], s.ln_eps)
    for rank, h, logits, t, uid in res:
        assert np.allclose(h, want, rtol=0, atol=1e-12)
        assert np.allclose(logits, want_logits, rtol=0, atol=1e-10)
        assert t == 1.5  # max over ranks of 0.5, 1.5
        assert uid == bytes(range(128))


def test_tp_slices_cover_the_model():
    cfg = ModelConfig(hidden=4096, n_heads=32, d_head=128, n_layers=32, d_mlp=16384, rotary_pct=0.25,
                      vocab=50432)
    for size in (1, 2, 4, 8):
        sl = [tp_slices(cfg, r, size) for r in range(size)]
        assert sl[0].heads[0] == 0 and sl[-1].heads[1] == 32
        assert all(a.heads[1] == b.heads[0] for a, b in zip(sl, sl[1:]))
        assert sl[-1].qkv_rows[1] == 3 * 4096 and sl[-1].out_cols[1] == 4096
        assert sl[-1].mlp_rows[1] == 16384 and sl[-1].vocab_rows[1] == 50432
        assert [x.root for x in sl] == [True] + [False] * (size - 1)
    with pytest.raises(ValueError, match="divide"):
        tp_slices(cfg, 0, 3)
