#!/usr/bin/env python
"""Small workload that touches every kernel family once, for compute-sanitizer
(memcheck / synccheck / racecheck / initcheck; tools/sanitize.sh):
  * the fused decode kernel: a C1-shape block step (BASELINE configs[0]) and
    two greedy decode steps of a 2-layer model with the LM head (cluster
    DSMEM exchanges, mbarrier ring, grid barriers, packed argmax);
  * the batched path: one B = 4 step (LN / RoPE / tiled attention / combine,
    the tcgen05 GEMM) and a 5-row prefill.
Checks the C1 block step against the oracle so a silent corruption fails."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import neox_oracle as O  # noqa: E402  (the checker)
from paper_2604_23553_b200 import Engine, ModelConfig  # noqa: E402


def main():
    cfg = ModelConfig(hidden=768, n_heads=12, d_head=64, n_layers=1, d_mlp=3072, rotary_pct=0.25, vocab=1000)
    s = O.Shape.of(cfg)
    rng = np.random.default_rng(0)
    pk = O.f16_round(rng.standard_normal((12, 128, 64)) * 0.5)
    pv = O.f16_round(rng.standard_normal((12, 128, 64)) * 0.5)
    x = rng.standard_normal(768) * 0.5
    with Engine(cfg, max_seq=256) as eng:
        eng.synth_block_weights(0, 0)
        eng.kv_write(0, 0, pk, pv)
        got = eng.block_step(0, 128, x)
    want = O.block_step(x, O.f16_params(O.synth_block(s, 0)), O.KV.of(pk, pv), 128, s)
    err = float(np.max(np.abs(got - want)) / np.max(np.abs(want)))
    print(f"C1 block step: scaled error {err:.3e}")
    assert err < 1e-4, err

    cfg2 = cfg.with_(n_layers=2)
    with Engine(cfg2, max_seq=64) as eng:
        eng.synth_model(0)
        eng.kv_synth_all(16, 3)
        toks = eng.generate(token=1, pos=16, steps=2, graph=False)
        print("greedy tokens", list(toks))
        eng.batch_init(4)
        eng.batch_kv_synth(16, 5)
        xs = rng.standard_normal((4, 768)) * 0.5
        hb, _ = eng.batch_forward(16, xs)
        print("batch forward", hb.shape)
        hp = eng.prefill(18, rng.standard_normal((5, 768)) * 0.5)
        print("prefill", np.asarray(hp).shape)
    # the reference's unit-level helpers on the GPU (csrc/nfb_split.cu)
    from paper_2604_23553_b200 import cluster as cl
    q, K, V = rng.standard_normal(80), rng.standard_normal((37, 80)), rng.standard_normal((37, 80))
    for red in (cl.RING, cl.TREE, cl.ReductionStrategy(cl.ReductionKind.PERMUTED_ATOMIC, 7)):
        for n in (1, 4, 64):
            o, _ = cl.attend_split(q, K, V, cl.ClusterSpec(n_blocks=n, reduction=red,
                                                           accumulation_precision=cl.Precision.FP16), 0.1)
            assert np.all(np.isfinite(o))
    y = cl.output_project_atomic(rng.standard_normal((4, 96)), rng.standard_normal((96, 96)), rng.standard_normal(96),
                                 rng.standard_normal(96), cl.ClusterSpec(n_blocks=4, accumulation_precision=cl.Precision.FP16,
                                                                         atomic_seed=3))
    print("split helpers", y.shape)
    print("sanitize workload done")


if __name__ == "__main__":
    main()
