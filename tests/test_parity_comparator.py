"""The parity comparator can fail (nf/verify.py:67-69, tests/test_verify.py:15-19
pattern): deliberately broken oracles at the smoke / C1 inputs must be
REJECTED by tests/parity.check, while fp32-level noise must pass."""

import math

import numpy as np
import pytest

from oracle import neox_oracle as O
from parity import TOL, check, scaled

S = O.Shape(hidden=768, n_heads=12, d_head=64, n_layers=1, d_mlp=3072, rotary_pct=0.25, vocab=1000)


def _inputs():
    rng = np.random.default_rng(0)
    pk = O.f16_round(rng.standard_normal((12, 128, 64)) * 0.5)
    pv = O.f16_round(rng.standard_normal((12, 128, 64)) * 0.5)
    x = rng.standard_normal(768) * 0.5
    return pk, pv, x, O.f16_params(O.synth_block(S, 0))


def _mutant(x, p, pk, pv, pos, s, bug):
    """oracle.block_step with one injected bug."""
    n1 = O.ln_two_pass(x, p["ln1_gain"], p["ln1_bias"], s.ln_eps)
    q, k, v = O.qkv_split(n1, p, s)
    q = O.rope(q, pos - 1 if bug == "rope_pos" else pos, s.rotary_dims, s.theta_base)
    if bug != "rope_key":
        k = O.rope(k, pos, s.rotary_dims, s.theta_base)
    d = s.d_head
    ctx = np.empty(s.hidden)
    for h in range(s.n_heads):
        keys = pk[h] if bug == "no_fresh" else np.concatenate([pk[h], k[h][None]])
        vals = pv[h] if bug == "no_fresh" else np.concatenate([pv[h], v[h][None]])
        scale = 1.0 / math.sqrt(d) if bug != "scale" else 1.0 / d
        ctx[h * d:(h + 1) * d] = O.attend(q[h], keys, vals, scale)
    if bug == "drop_head":
        ctx[:d] = 0.0
    attn = x + p["out_weight"] @ ctx + p["out_bias"]
    n2 = O.ln_two_pass(x, p["ln2_gain"], p["ln2_bias"], s.ln_eps)
    kind = "exact" if bug == "gelu" else "tanh"
    mlp = O.mlp(n2, p, kind)
    if bug == "no_down_bias":
        mlp = mlp - p["down_bias"]
    return attn + mlp


BUGS = ["drop_head", "no_fresh", "rope_key", "rope_pos", "scale", "gelu", "no_down_bias"]


def test_unmutated_oracle_and_fp32_noise_pass():
    pk, pv, x, p = _inputs()
    want = O.block_step(x, p, O.KV.of(pk, pv), 128, S)
    assert np.max(np.abs(_mutant(x, p, pk, pv, 128, S, None) - want)) <= 1e-12
    fp32 = want.astype(np.float32).astype(np.float64) * (1 + 3e-7)
    check(fp32, want, x)


@pytest.mark.parametrize("bug", BUGS)
def test_comparator_rejects_mutation(bug):
    pk, pv, x, p = _inputs()
    want = O.block_step(x, p, O.KV.of(pk, pv), 128, S)
    bad = _mutant(x, p, pk, pv, 128, S, bug)
    with pytest.raises(AssertionError):
        check(bad, want, x, what=bug)


def test_north_star_bar_alone_would_miss_some_mutations():
    """Documents why the regression guard exists: the 2e-2 bar on the block
    output passes several of these bugs."""
    pk, pv, x, p = _inputs()
    want = O.block_step(x, p, O.KV.of(pk, pv), 128, S)
    missed = [b for b in BUGS if scaled(_mutant(x, p, pk, pv, 128, S, b), want) <= TOL]
    assert {"drop_head", "no_fresh", "rope_key"} <= set(missed)
