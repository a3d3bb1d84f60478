"""Generate the golden fixtures under tests/golden/ by importing the REFERENCE.

Run in the build container (the reference is mounted read-only at
/root/reference; it does not exist on the GPU box):

    python tests/golden/make_golden.py

Every number in the fixtures comes from the reference package ``neoxfuse``
itself (``/root/reference/pkg/src/neoxfuse``).  The fixtures pin the CPU
oracle (``oracle/neox_oracle.py``) -- see ``tests/test_oracle_golden.py`` --
and, through the oracle, the GPU parity tests.
"""

import json
import os
import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF = os.environ.get("NEOXFUSE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

import neoxfuse as nf  # noqa: E402
from neoxfuse import halfnum  # noqa: E402
from neoxfuse.cluster import ClusterSpec, fused_block_step  # noqa: E402
from neoxfuse.config import ModelConfig, preset  # noqa: E402
from neoxfuse.golden import decoder_block_golden  # noqa: E402
from neoxfuse.plans import plan_baseline, plan_full_fused, kernel_layer_bytes  # noqa: E402
from neoxfuse.weights import KVCache, synth_weights, TENSOR_NAMES  # noqa: E402

OUT = Path(__file__).resolve().parent

C1 = dict(hidden=768, n_heads=12, d_head=64, n_layers=12, d_mlp=3072,
          rotary_pct=0.25, vocab=50304)
D80 = dict(hidden=1280, n_heads=16, d_head=80, n_layers=1, d_mlp=5120,
           rotary_pct=0.25, vocab=512)
SEQ = dict(hidden=512, n_heads=8, d_head=64, n_layers=1, d_mlp=2048,
           rotary_pct=0.25, vocab=256, parallel_residual=False)


def f16(w):
    """Round every tensor of a BlockWeights through binary16 (reference RNE)."""
    return nf.BlockWeights(**{n: halfnum.half_round_array(getattr(w, n))
                              for n in TENSOR_NAMES})


def prng():
    seeds = np.array([0, 1, 12345, (1 << 63) + 5, (1 << 64) - 1], dtype=np.uint64)
    counters = np.concatenate([
        np.arange(64, dtype=np.uint64),
        (np.uint64(7) << np.uint64(32)) + np.arange(64, dtype=np.uint64),
        np.array([(1 << 40) + 3, (11 << 32) + 123456789], dtype=np.uint64),
    ])
    draws = np.stack([halfnum.counter_rand_u64_array(int(s), counters) for s in seeds])
    scalar = np.array([halfnum.counter_rand_u64(int(seeds[2]), int(c)) for c in counters[:8]],
                      dtype=np.uint64)
    np.savez(OUT / "prng.npz", seeds=seeds, counters=counters, draws=draws, scalar=scalar)


def half():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(4000) * 10.0 ** rng.integers(-9, 6, 4000),
        # exact binary16 ties and neighbours, subnormal range, overflow edge
        (np.arange(-2048, 2048) + 0.5) * 2.0 ** -10,
        (np.arange(0, 512) + 0.5) * 2.0 ** -24,
        np.array([65504.0, 65519.99, 65520.0, 1e6, -1e6, 0.0, -0.0, 2.0 ** -25,
                  2.0 ** -25 * 1.0000001, 2.0 ** -26, 6.1e-5, 5.96e-8]),
    ])
    np.savez(OUT / "half.npz", x=x, y=halfnum.half_round_array(x),
             bits=np.array([halfnum.half_round(v).bits for v in x[:64]]))


def synth():
    out = {}
    rng = np.random.default_rng(1)
    for tag, cfg, seed in (("tiny", preset("tiny"), 5), ("c1", ModelConfig(**C1), 0),
                           ("d80", ModelConfig(**D80), 3)):
        w = synth_weights(cfg, seed)
        for n in TENSOR_NAMES:
            a = getattr(w, n).ravel()
            idx = rng.integers(0, a.size, 64)
            out[f"{tag}.{n}.sum"] = np.array(np.sum(a))
            out[f"{tag}.{n}.idx"] = idx
            out[f"{tag}.{n}.val"] = a[idx]
            out[f"{tag}.{n}.head"] = a[:16]
            out[f"{tag}.{n}.tail"] = a[-16:]
            out[f"{tag}.{n}.f16sum"] = np.array(np.sum(halfnum.half_round_array(a)))
    np.savez(OUT / "synth.npz", **out)


def _prefix(rng, cfg, n):
    pk = rng.standard_normal((cfg.n_heads, n, cfg.d_head)) * 0.5
    pv = rng.standard_normal((cfg.n_heads, n, cfg.d_head)) * 0.5
    return halfnum.half_round_array(pk), halfnum.half_round_array(pv)


def blocks():
    """decoder_block_golden / fused_block_step runs on fp16-rounded weights.

    Input recipe (re-created by the tests): rng = default_rng(seed);
    prefix K, V = N(0,1)*0.5 [H, prefix, d] rounded to fp16; then per step
    x_t = N(0,1)*0.5 [hidden]."""
    cases = {
        "c1": (ModelConfig(**C1), 0, 128, 1, "tanh"),
        "c1exact": (ModelConfig(**C1), 0, 128, 1, "exact"),
        "d80": (ModelConfig(**D80), 3, 40, 3, "tanh"),
        "seq": (ModelConfig(**SEQ), 4, 17, 2, "exact"),
        "p0": (ModelConfig(**C1), 6, 0, 3, "tanh"),
        "wide": (preset("pythia-2.8b").with_(n_layers=1), 9, 3, 1, "tanh"),
    }
    for tag, (cfg, seed, npre, steps, gelu) in cases.items():
        w = f16(synth_weights(cfg, seed))
        rng = np.random.default_rng(seed)
        pk, pv = _prefix(rng, cfg, npre)
        xs = rng.standard_normal((steps, cfg.hidden)) * 0.5
        cache = KVCache.from_arrays(pk, pv) if npre else KVCache(cfg.n_heads, cfg.d_head)
        fcache = KVCache.from_arrays(pk, pv) if npre else KVCache(cfg.n_heads, cfg.d_head)
        outs, fouts = [], []
        for t in range(steps):
            outs.append(decoder_block_golden(xs[t], w, cache, npre + t, cfg, gelu))
            o, tr = fused_block_step(xs[t], w, fcache, npre + t, cfg, ClusterSpec(n_blocks=4),
                                     plan_full_fused(), gelu)
            fouts.append(o)
        keys, vals = cache.keys(), cache.values()
        np.savez(OUT / f"block_{tag}.npz", seed=seed, prefix=npre, steps=steps,
                 gelu=gelu, model=json.dumps({k: getattr(cfg, k) for k in (
                     "hidden", "n_heads", "d_head", "n_layers", "d_mlp", "rotary_pct",
                     "vocab", "ln_eps", "theta_base", "parallel_residual")}),
                 xs=xs, outs=np.array(outs), fused=np.array(fouts),
                 new_keys=keys[:, npre:], new_values=vals[:, npre:],
                 trace_offchip=tr.bytes_offchip, trace_onchip=tr.bytes_onchip,
                 trace_sync=tr.sync_steps, trace_dsmem=tr.dsmem_exchanges)


def fidelity():
    out = {}
    for seed in range(3):
        inst = nf.synthetic_instance(seed)
        out[f"syn{seed}.golden"] = inst.golden_logits()
        out[f"syn{seed}.exact"] = inst.variant_logits(ClusterSpec(n_blocks=4))
    adv = nf.adversarial_instance()
    out["adv.golden"] = adv.golden_logits()
    # a 160M-shape probe instance: 1 block, prompt 16, 6 teacher-forced steps
    cfg = ModelConfig(**C1).with_(n_layers=1, vocab=1000)
    inst = nf.synthetic_instance(21, cfg, prompt_len=16, steps=6)
    out["c1probe.golden"] = inst.golden_logits()
    rep = nf.compare(out["syn0.golden"], out["syn0.golden"] + np.linspace(0, 1e-3, 11))
    out["compare.syn0"] = np.array([rep.token_match_rate, rep.logits_mae,
                                    rep.topk_agreement[5], rep.topk_agreement[10]])
    np.savez(OUT / "fidelity.npz", **out)


def bytes_model():
    doc = {}
    for name, cfg in (("pythia-2.8b", preset("pythia-2.8b")), ("pythia-6.9b", preset("pythia-6.9b")),
                      ("c1", ModelConfig(**C1).with_(n_layers=1))):
        for P in (1, 129, 1025, 1152, 2049, 4097):
            tr = nf.traffic(plan_full_fused(), cfg, P)
            doc[f"{name}.full.{P}"] = [tr.layer_bytes, tr.lm_head_bytes, tr.step_bytes]
            doc[f"{name}.baseline.{P}"] = kernel_layer_bytes(plan_baseline(), cfg, P)
        pc = nf.count_params(cfg)
        doc[f"{name}.params"] = [pc.per_layer, pc.blocks, pc.final_ln, pc.unembedding]
        doc[f"{name}.flops.1024"] = nf.flops_per_token(cfg, 1024)
    doc["mlp_saving.2.8b"] = nf.mlp_fusion_saving_bytes(preset("pythia-2.8b"))
    (OUT / "bytes.json").write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")


def cli_fixture():
    """The reference CLI's own golden fixture (`neoxfuse golden`, nf/cli.py:343-397)
    for a 256-hidden, d_head 64 block: the JSON parity artefact the B200 path
    replays (paper_2604_23553_b200.formats.replay_golden_fixture)."""
    import argparse
    from neoxfuse import cli
    cfg = OUT / "_cli_fixture.cfg"
    cfg.write_text("model.hidden=256\nmodel.n_heads=4\nmodel.d_head=64\nmodel.n_layers=1\n"
                   "model.d_mlp=1024\nmodel.rotary_pct=0.25\nmodel.vocab=64\nrun.gelu=tanh\n")
    try:
        ns = argparse.Namespace(config=str(cfg), preset=None, out=str(OUT / "cli_golden_h256.json"),
                                format="json", seed=21, seq_lens=None, steps=6)
        cli.cmd_golden(ns)
    finally:
        cfg.unlink()


def prefill():
    """prefill_attention_tiled (nf/golden.py:234-265): causal and full
    attention of one head over a 37-position sequence, several tile sizes."""
    from neoxfuse.golden import prefill_attention_tiled
    rng = np.random.default_rng(31)
    out = {}
    for tag, d in (("d80", 80), ("d64", 64)):
        Q, K, V = (rng.standard_normal((37, d)) * 0.7 for _ in range(3))
        out[f"{tag}.Q"], out[f"{tag}.K"], out[f"{tag}.V"] = Q, K, V
        for tile in (1, 5, 16, 37):
            out[f"{tag}.causal.{tile}"] = prefill_attention_tiled(Q, K, V, tile)
            out[f"{tag}.full.{tile}"] = prefill_attention_tiled(Q, K, V, tile, causal=False)
    np.savez(OUT / "prefill.npz", **out)


def split():
    """attend_split and output_project_atomic (nf/cluster.py:211-285): one
    head's split-KV attention under every merge order / precision, and the
    atomic output projection, exact and FP16-atomic, over several seeds."""
    import warnings
    from neoxfuse.cluster import attend_split, output_project_atomic
    from neoxfuse.halfnum import RING, TREE, Precision, permuted_atomic
    rng = np.random.default_rng(47)
    out = {}
    strategies = {"ring": RING, "tree": TREE, "perm7": permuted_atomic(7), "perm123": permuted_atomic(123)}
    for d, seq in ((64, 1), (80, 5), (64, 37), (80, 300)):
        tag = f"d{d}s{seq}"
        q = rng.standard_normal(d) * 0.8
        K = rng.standard_normal((seq, d)) * 0.8
        V = rng.standard_normal((seq, d))
        out[f"{tag}.q"], out[f"{tag}.K"], out[f"{tag}.V"] = q, K, V
        for n in (1, 2, 3, 4, 8, 16):
            for sname, strat in strategies.items():
                for prec in (Precision.EXACT, Precision.FP16):
                    spec = ClusterSpec(n_blocks=n, reduction=strat, accumulation_precision=prec)
                    with warnings.catch_warnings():
                        warnings.simplefilter("ignore", RuntimeWarning)
                        o, tr = attend_split(q, K, V, spec, 1.0 / np.sqrt(d))
                    key = f"{tag}.n{n}.{sname}.{prec.value}"
                    out[key + ".out"] = o
                    r = tr.records[0]
                    out[key + ".trace"] = np.array([r.bytes_offchip, r.bytes_onchip, r.sync_steps,
                                                    r.dsmem_exchanges])
    for hidden, n in ((64, 1), (64, 3), (96, 4), (128, 8), (80, 16)):
        tag = f"h{hidden}n{n}"
        P = rng.standard_normal((n, hidden)) * 2.0
        W = rng.standard_normal((hidden, hidden)) * 0.3
        b = rng.standard_normal(hidden) * 0.5
        res = rng.standard_normal(hidden) * 4.0
        out[f"{tag}.P"], out[f"{tag}.W"], out[f"{tag}.b"], out[f"{tag}.res"] = P, W, b, res
        for prec in (Precision.EXACT, Precision.FP16):
            for seed in (0, 5, 2**40 + 3):
                spec = ClusterSpec(n_blocks=n, accumulation_precision=prec, atomic_seed=seed)
                out[f"{tag}.{prec.value}.{seed}"] = output_project_atomic(P, W, b, res, spec)
    np.savez(OUT / "split.npz", **out)


ALL = [cli_fixture, prng, half, synth, blocks, fidelity, bytes_model, prefill, split]

if __name__ == "__main__":
    # python tests/golden/make_golden.py [name ...]  (default: every fixture)
    pick = sys.argv[1:]
    for fn in ALL:
        if not pick or fn.__name__ in pick:
            fn()
    print("golden fixtures written to", OUT)
