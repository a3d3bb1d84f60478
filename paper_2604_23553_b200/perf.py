"""Roofline arithmetic: algorithmic bytes and FLOPs per decode step.

Mirror of the reference's traffic / parameter / FLOP accounting
(nf/perfmodel.py:96-121, 261-292).  These are the numerators of the
``roofline`` object bench.py reports; the denominators are the measured B200
peaks in MEASURED_PEAKS.json.  (The reference's analytic RTX-5090 timing
model -- HardwareModel / step_time / calibrate -- is out of scope: this build
measures instead of modelling.)
"""

from __future__ import annotations

from dataclasses import dataclass

from .plans import FusionPlan, kernel_layer_bytes, plan_full_fused

DEFAULT_ELEM_SIZE = 2


@dataclass
class TrafficReport:
    plan_name: str
    seq_len: int
    elem_size: int
    per_kernel_layer_bytes: list
    layer_bytes: int
    lm_head_bytes: int
    step_bytes: int


def lm_head_bytes(cfg, elem_size: int = DEFAULT_ELEM_SIZE) -> int:
    """Final LN params + unembedding matrix, streamed once per step."""
    return (2 + cfg.vocab) * cfg.hidden * elem_size


def traffic(plan: FusionPlan, cfg, seq_len: int, elem_size: int = DEFAULT_ELEM_SIZE) -> TrafficReport:
    per = kernel_layer_bytes(plan, cfg, seq_len, elem_size)
    layer = sum(per)
    head = lm_head_bytes(cfg, elem_size)
    return TrafficReport(plan.name or "custom", seq_len, elem_size,
                         [(k.name, b) for k, b in zip(plan.kernels, per)],
                         layer, head, cfg.n_layers * layer + head)


def step_bytes(cfg, seq_len: int, elem_size: int = DEFAULT_ELEM_SIZE, head: bool = True) -> int:
    """Bytes of one fully fused decode step at KV length seq_len (= P)."""
    t = traffic(plan_full_fused(), cfg, seq_len, elem_size)
    return t.step_bytes if head else t.step_bytes - t.lm_head_bytes


def mean_step_bytes(cfg, first_pos: int, steps: int, head: bool = True) -> float:
    """Mean bytes over decode positions first_pos .. first_pos+steps-1 (P = pos+1)."""
    return sum(step_bytes(cfg, p + 1, head=head) for p in range(first_pos, first_pos + steps)) / steps


@dataclass
class ParamCounts:
    per_layer: int
    blocks: int
    final_ln: int
    unembedding: int
    non_embedding: int


def count_params(cfg) -> ParamCounts:
    h, m = cfg.hidden, cfg.d_mlp
    per_layer = 4 * h + 3 * h * (h + 1) + h * (h + 1) + m * (h + 1) + h * (m + 1)
    blocks = per_layer * cfg.n_layers
    return ParamCounts(per_layer, blocks, 2 * h, cfg.vocab * h, blocks + 2 * h)


def flops_per_token(cfg, position: int) -> float:
    """2 FLOPs per weight MAC + 4*h*(position+1) attention FLOPs per layer."""
    c = count_params(cfg)
    return 2.0 * (c.non_embedding + c.unembedding) + 4.0 * cfg.hidden * cfg.n_layers * (position + 1)


def batch_step_bytes(cfg, seq_len: int, batch: int, elem_size: int = DEFAULT_ELEM_SIZE) -> int:
    """Algorithmic bytes of one batched decode step (configs[3]): the weights
    and LM head once, the KV history (read 2*P*h, write 2*h per layer) and the
    residual stream per sequence -- SURVEY.md §8(d) batch extension
    ``weights_once + B * (KV(P) + activations)``."""
    one = step_bytes(cfg, seq_len, elem_size)
    h, L = cfg.hidden, cfg.n_layers
    per_seq = L * (2 * seq_len * h * elem_size + 2 * h * elem_size + 2 * h * 4)
    return one + (batch - 1) * per_seq


def mean_batch_step_bytes(cfg, first_pos: int, steps: int, batch: int) -> float:
    return sum(batch_step_bytes(cfg, p + 1, batch) for p in range(first_pos, first_pos + steps)) / steps
