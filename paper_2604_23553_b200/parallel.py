"""Multi-GPU plumbing: the tensor-parallel shard plan and the few collectives
the host needs (torch.distributed, NCCL on GPUs or gloo in CPU tests).

Data parallel (BASELINE.json configs[4]): independent decode streams, one
``Engine`` per GPU, no data-path collective; only the timing is reduced
(max over ranks).  Tensor parallel (configs[2], Pythia-6.9B): heads, FFN rows
and vocabulary are split over the ranks exactly as ``tp_slices`` says -- the
C library (csrc/nfb_api.cu, nfb_create_tp / nfb_synth_block_weights) applies
the same slices -- and the layer output is the sum over ranks of each rank's
split-K partial, rank 0 adding the residual and the biases (one all-reduce
per layer thanks to the parallel residual, nf/golden.py:224-228).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class TPSlices:
    heads: tuple[int, int]        # attention heads [hs, he)
    qkv_rows: tuple[int, int]     # rows of W_qkv / b_qkv (interleaved per head, nf/weights.py:3-5)
    out_cols: tuple[int, int]     # columns of W_out (context elements of the heads)
    mlp_rows: tuple[int, int]     # rows of W_up / b_up, columns of W_down
    vocab_rows: tuple[int, int]   # rows of the unembedding (vocab-parallel LM head)
    root: bool                    # adds residual + b_out + b_down in the layer sum


def tp_slices(cfg, rank: int, size: int) -> TPSlices:
    """Shard ``rank`` of ``size`` of a model config (raises on uneven splits,
    like nfb_create_tp)."""
    if size < 1 or not 0 <= rank < size:
        raise ValueError("bad tensor-parallel rank / size")
    for name in ("n_heads", "d_mlp", "vocab"):
        if getattr(cfg, name) % size:
            raise ValueError(f"{name} must divide by the tensor-parallel size")
    if size > 1 and not cfg.parallel_residual:
        raise ValueError("tensor parallelism needs the parallel residual (one all-reduce per layer)")
    H, d, m, V = cfg.n_heads // size, cfg.d_head, cfg.d_mlp // size, cfg.vocab // size
    hs, he = rank * H, (rank + 1) * H
    return TPSlices(heads=(hs, he), qkv_rows=(hs * 3 * d, he * 3 * d), out_cols=(hs * d, he * d),
                    mlp_rows=(rank * m, (rank + 1) * m), vocab_rows=(rank * V, (rank + 1) * V),
                    root=rank == 0)


def world():
    """(world_size, rank) of the default process group, (1, 0) without one."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def max_over_ranks(x: float, device=None) -> float:
    """Device-timed seconds -> the max over ranks (the bench contract)."""
    import torch
    import torch.distributed as dist
    n, _ = world()
    if n == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def broadcast_bytes(b: bytes | None, nbytes: int, src: int = 0, device=None) -> bytes:
    """Share ``nbytes`` (e.g. the 128-byte NCCL unique id) from ``src``."""
    import torch
    import torch.distributed as dist
    n, rank = world()
    if n == 1:
        return bytes(b)
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if rank == src:
        buf.copy_(torch.frombuffer(bytearray(b), dtype=torch.uint8))
    dist.broadcast(buf, src)
    return bytes(buf.cpu().numpy().tobytes())
