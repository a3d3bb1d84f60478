"""CPU oracle for the GPT-NeoX single-token decode block -- TEST INFRASTRUCTURE.

This module is the *checker*, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import it.  The shipped decode path (``paper_2604_23553_b200``) runs the
sm_100a kernels through the C-ABI library and fails loudly when that library
is missing; it never routes through this file.

It is a float64 numpy restatement of the reference package ``neoxfuse``
(``/root/reference/pkg/src/neoxfuse``, abbreviated ``nf/`` below).  Each
function cites the reference lines it follows.  Parity of this restatement is
PINNED against golden vectors produced by importing the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``; checked by
``tests/test_oracle_golden.py``): SplitMix64 draws and synthesized weights
bit-exact, binary16 rounding bit-exact, block outputs / caches / fused-step
outputs to <= 1e-12, byte-model integers exact.

Third-party arithmetic: numpy matmul (OpenBLAS) and ``scipy.special.erf``
(GELU exact) are the same libraries the reference calls (``nf/golden.py:19-20``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_MASK64 = (1 << 64) - 1
_GOLDEN_GAMMA = 0x9E3779B97F4A7C15

# Tensor order of a block; fixes the PRNG stream index of each tensor
# (nf/weights.py:55 -- dataclass field order of BlockWeights, nf/weights.py:24-37).
BLOCK_TENSORS = (
    "ln1_gain", "ln1_bias", "qkv_weight", "qkv_bias", "out_weight", "out_bias",
    "ln2_gain", "ln2_bias", "up_weight", "up_bias", "down_weight", "down_bias",
)


# ---------------------------------------------------------------------------
# Shapes (nf/config.py:11-49).

@dataclass(frozen=True)
class Shape:
    hidden: int
    n_heads: int
    d_head: int
    n_layers: int
    d_mlp: int
    rotary_pct: float
    vocab: int
    ln_eps: float = 1e-5
    theta_base: float = 10000.0
    parallel_residual: bool = True

    @property
    def rotary_dims(self) -> int:  # nf/config.py:44-46
        return math.floor(self.rotary_pct * self.d_head)

    @classmethod
    def of(cls, cfg) -> "Shape":
        return cls(cfg.hidden, cfg.n_heads, cfg.d_head, cfg.n_layers, cfg.d_mlp,
                   cfg.rotary_pct, cfg.vocab, cfg.ln_eps, cfg.theta_base,
                   cfg.parallel_residual)


# ---------------------------------------------------------------------------
# Counter PRNG and weight synthesis.

def splitmix64(seed: int, counters) -> np.ndarray:
    """SplitMix64 output function of seed + (c+1)*gamma (nf/halfnum.py:35-59)."""
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _MASK64) + (c + np.uint64(1)) * np.uint64(_GOLDEN_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform_stream(seed: int, stream: int, n: int) -> np.ndarray:
    """n doubles in [-1, 1): (u >> 11) * 2^-52 - 1 (nf/weights.py:58-62)."""
    counters = np.uint64(stream << 32) + np.arange(n, dtype=np.uint64)
    u = splitmix64(seed, counters)
    return (u >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0


def block_shapes(s: Shape) -> dict:
    h, m = s.hidden, s.d_mlp
    return {
        "ln1_gain": (h,), "ln1_bias": (h,),
        "qkv_weight": (3 * h, h), "qkv_bias": (3 * h,),
        "out_weight": (h, h), "out_bias": (h,),
        "ln2_gain": (h,), "ln2_bias": (h,),
        "up_weight": (m, h), "up_bias": (m,),
        "down_weight": (h, m), "down_bias": (h,),
    }


def synth_block(s: Shape, seed: int) -> dict:
    """Deterministic block parameters (nf/weights.py:65-94): projections
    u/sqrt(fan_in), LN gains 1+0.1u, LN biases 0.1u, other biases 0.02u."""
    out = {}
    for stream, (name, shape) in enumerate(
            (n, block_shapes(s)[n]) for n in BLOCK_TENSORS):
        u = uniform_stream(seed, stream, int(np.prod(shape))).reshape(shape)
        if name.endswith("_weight"):
            out[name] = u / np.sqrt(shape[1])
        elif name.endswith("gain"):
            out[name] = 1.0 + 0.1 * u
        elif name in ("ln1_bias", "ln2_bias"):
            out[name] = 0.1 * u
        else:
            out[name] = 0.02 * u
    return out


# Model-level extras that the reference lacks: embedding, final
# LN and LM head.  Documented recipe: seed
# head_seed(base, n_layers) = base + n_layers (never a layer seed), streams
# 0..3 = embed [V,h] u, lnf_gain 1+0.1u, lnf_bias 0.1u, unembed [V,h] u/sqrt(h).
HEAD_TENSORS = ("embed", "lnf_gain", "lnf_bias", "unembed")


def layer_seed(base: int, layer: int) -> int:
    return (base + layer) & _MASK64


def head_seed(base: int, n_layers: int) -> int:
    return (base + n_layers) & _MASK64


def synth_head(s: Shape, seed: int) -> dict:
    h, V = s.hidden, s.vocab
    return {
        "embed": uniform_stream(seed, 0, V * h).reshape(V, h),
        "lnf_gain": 1.0 + 0.1 * uniform_stream(seed, 1, h),
        "lnf_bias": 0.1 * uniform_stream(seed, 2, h),
        "unembed": uniform_stream(seed, 3, V * h).reshape(V, h) / np.sqrt(h),
    }


def f16_round(x) -> np.ndarray:
    """Round float64 -> nearest binary16 (ties to even, overflow to inf) and
    back to float64 (nf/halfnum.py:165-220).  numpy's direct double->half
    cast is correctly rounded; pinned bit-exact against the reference's
    integer algorithm by the golden vectors."""
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)


def f16_params(p: dict) -> dict:
    """What the GPU sees: every parameter stored as binary16."""
    return {k: f16_round(v) for k, v in p.items()}


# ---------------------------------------------------------------------------
# Block operators (nf/golden.py).

def _finite(x):
    if not np.all(np.isfinite(x)):  # nf/golden.py:29-31
        raise ValueError("non-finite activation")


def ln_two_pass(x, g, b, eps):
    """nf/golden.py:34-40."""
    x = np.asarray(x, dtype=np.float64)
    _finite(x)
    mu = x.mean()
    var = np.mean((x - mu) ** 2)
    return (x - mu) / np.sqrt(var + eps) * g + b


def ln_single_pass(x, g, b, eps):
    """nf/golden.py:43-49 (fused path's one-sweep moments, clamped)."""
    x = np.asarray(x, dtype=np.float64)
    _finite(x)
    mu = x.mean()
    var = max(np.mean(x * x) - mu * mu, 0.0)
    return (x - mu) / np.sqrt(var + eps) * g + b


def qkv_split(xn, p, s: Shape):
    """Interleaved per-head rows Q|K|V (nf/golden.py:55-65)."""
    y = p["qkv_weight"] @ np.asarray(xn, dtype=np.float64) + p["qkv_bias"]
    d = s.d_head
    y = y.reshape(s.n_heads, 3 * d)
    return y[:, :d].copy(), y[:, d:2 * d].copy(), y[:, 2 * d:].copy()


def rope(v, pos, rd, base=10000.0):
    """Rotate pairs (i, i+rd/2); dims >= rd pass through (nf/golden.py:68-92)."""
    v = np.asarray(v, dtype=np.float64)
    if rd < 2 or rd % 2:
        raise ValueError("rotary_dims must be an even number >= 2")
    if rd > v.shape[-1]:
        raise ValueError("rotary_dims exceeds head size")
    half = rd // 2
    theta = pos * base ** (-2.0 * np.arange(half, dtype=np.float64) / rd)
    c, sn = np.cos(theta), np.sin(theta)
    out = v.copy()
    a, b = v[..., :half], v[..., half:rd]
    out[..., :half] = a * c - b * sn
    out[..., half:rd] = a * sn + b * c
    return out


def sm_state(q, keys, values, scale):
    """(m, l, o) of one contiguous KV slice (nf/golden.py:116-125)."""
    keys = np.asarray(keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    if keys.shape[0] == 0:
        return (-math.inf, 0.0, np.zeros(values.shape[-1]))
    logits = keys @ np.asarray(q, dtype=np.float64) * scale
    m = float(np.max(logits))
    w = np.exp(logits - m)
    return (m, float(np.sum(w)), w @ values)


def sm_merge(a, b):
    """LSE merge; empty states are identities (nf/golden.py:128-136)."""
    if a[1] == 0.0:
        return (b[0], b[1], b[2].copy())
    if b[1] == 0.0:
        return (a[0], a[1], a[2].copy())
    m = max(a[0], b[0])
    fa, fb = math.exp(a[0] - m), math.exp(b[0] - m)
    return (m, a[1] * fa + b[1] * fb, a[2] * fa + b[2] * fb)


def attend(q, keys, values, scale):
    """nf/golden.py:139-150."""
    if np.asarray(keys).shape[0] == 0:
        raise ValueError("attention over empty cache")
    m, l, o = sm_state(q, keys, values, scale)
    if l == 0.0:
        raise ValueError("empty attention state")
    return o / l


def gelu(x, kind="tanh"):
    """nf/golden.py:156-169."""
    x = np.asarray(x, dtype=np.float64)
    if kind == "tanh":
        return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))
    if kind == "exact":
        from scipy.special import erf
        return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))
    raise ValueError(f"unknown gelu variant {kind!r} (use 'exact' or 'tanh')")


def mlp(xn, p, kind="tanh"):
    """nf/golden.py:172-179."""
    hdn = p["up_weight"] @ np.asarray(xn, dtype=np.float64) + p["up_bias"]
    return p["down_weight"] @ gelu(hdn, kind) + p["down_bias"]


class KV:
    """Append-only per-head history, keys post-rotation (nf/weights.py:132-183).
    Preallocated instead of capacity doubling; same observable behaviour."""

    def __init__(self, n_heads, d_head, cap=16):
        self.k = np.zeros((n_heads, cap, d_head))
        self.v = np.zeros((n_heads, cap, d_head))
        self.n = 0

    @classmethod
    def of(cls, keys, values):
        keys = np.asarray(keys, dtype=np.float64)
        values = np.asarray(values, dtype=np.float64)
        c = cls(keys.shape[0], keys.shape[2], max(16, keys.shape[1] + 256))
        c.k[:, :keys.shape[1]] = keys
        c.v[:, :keys.shape[1]] = values
        c.n = keys.shape[1]
        return c

    def __len__(self):
        return self.n

    def append(self, k, v):
        if self.n == self.k.shape[1]:
            grow = self.k.shape[1]
            self.k = np.concatenate([self.k, np.zeros_like(self.k[:, :grow])], 1)
            self.v = np.concatenate([self.v, np.zeros_like(self.v[:, :grow])], 1)
        self.k[:, self.n] = k
        self.v[:, self.n] = v
        self.n += 1

    def head(self, h):
        return self.k[h, :self.n], self.v[h, :self.n]

    def keys(self):
        return self.k[:, :self.n].copy()

    def values(self):
        return self.v[:, :self.n].copy()


def block_step(x, p, cache, pos, s: Shape, kind="tanh", ln=ln_two_pass, kv_store=None):
    """One decode step of the block, appending this step's K/V
    (nf/golden.py:189-228; with ``ln=ln_single_pass`` the numerics of
    nf/cluster.py:316,351 in EXACT mode).

    ``kv_store`` (default None = the reference: K/V kept in float64) is applied
    to the K/V *stored* in the cache -- ``f16_round`` restates the device's
    fp16 KV cache.  The current token still attends with its exact K/V (the
    fused kernel keeps them in fp32 registers); only later steps see the
    stored values."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (s.hidden,):
        raise ValueError(f"input must have shape ({s.hidden},)")
    if len(cache) != pos:
        raise ValueError(f"cache holds {len(cache)} positions, expected {pos}")
    n1 = ln(x, p["ln1_gain"], p["ln1_bias"], s.ln_eps)
    q, k, v = qkv_split(n1, p, s)
    q = rope(q, pos, s.rotary_dims, s.theta_base)
    k = rope(k, pos, s.rotary_dims, s.theta_base)
    cache.append(kv_store(k) if kv_store else k, kv_store(v) if kv_store else v)
    scale = 1.0 / math.sqrt(s.d_head)  # nf/golden.py:185-186
    ctx = np.empty(s.hidden)
    d = s.d_head
    for h in range(s.n_heads):
        kh, vh = cache.head(h)
        if kv_store:
            kh, vh = kh.copy(), vh.copy()
            kh[-1], vh[-1] = k[h], v[h]
        ctx[h * d:(h + 1) * d] = attend(q[h], kh, vh, scale)
    attn_res = x + p["out_weight"] @ ctx + p["out_bias"]
    ln2_in = x if s.parallel_residual else attn_res
    n2 = ln(ln2_in, p["ln2_gain"], p["ln2_bias"], s.ln_eps)
    return attn_res + mlp(n2, p, kind)


def prefill_attention(Q, K, V, tile, causal=True, scale=None, prefix_keys=None, prefix_values=None):
    """Causal attention over a sequence, keys folded in tiles of ``tile``
    positions into a running softmax state per query row
    (``prefill_attention_tiled``, nf/golden.py:234-265).  Extension used by
    the prefill path: an optional cached prefix [P0, d] that every query row
    sees before the sequence (row i then sees P0 + i + 1 keys when causal);
    with no prefix this is exactly the reference function."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    if Q.ndim != 2 or K.shape != Q.shape or V.shape != Q.shape:
        raise ValueError("Q, K, V must share shape [seq, d_head]")
    if tile < 1:
        raise ValueError("tile must be >= 1")
    seq, d = Q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    if prefix_keys is not None:
        K = np.concatenate([np.asarray(prefix_keys, np.float64), K])
        V = np.concatenate([np.asarray(prefix_values, np.float64), V])
    p0 = K.shape[0] - seq
    out = np.empty((seq, d))
    for i in range(seq):
        limit = p0 + i + 1 if causal else K.shape[0]
        st = (-math.inf, 0.0, np.zeros(d))
        for t0 in range(0, limit, tile):
            t1 = min(t0 + tile, limit)
            st = sm_merge(st, sm_state(Q[i], K[t0:t1], V[t0:t1], scale))
        out[i] = st[2] / st[1]
    return out


def causal_attention(Q, K, V, scale):
    """Vectorised form of ``prefill_attention`` for query rows that are the
    LAST seq rows of K/V (row i sees keys [0, P0 + i]): Q [H, T, d], K/V
    [H, P0 + T, d] -> [H, T, d].  One softmax per row instead of the tiled
    fold (equal to it up to float64 merge order; pinned in tests)."""
    Q = np.asarray(Q, np.float64)
    H, T, d = Q.shape
    P = K.shape[1]
    S = np.einsum("htd,hpd->htp", Q, K) * scale
    mask = np.arange(P)[None, :] > (P - T + np.arange(T))[:, None]
    S = np.where(mask[None], -np.inf, S)
    m = S.max(axis=2, keepdims=True)
    w = np.exp(S - m)
    return np.einsum("htp,hpd->htd", w, V) / w.sum(axis=2, keepdims=True)


def rope_rows(v, positions, rd, base=10000.0):
    """``rope`` with one position per row: v [T, ..., d], positions [T]."""
    v = np.asarray(v, dtype=np.float64)
    half = rd // 2
    theta = np.asarray(positions, np.float64)[:, None] * base ** (-2.0 * np.arange(half, dtype=np.float64) / rd)
    shape = (v.shape[0],) + (1,) * (v.ndim - 2) + (half,)
    c, sn = np.cos(theta).reshape(shape), np.sin(theta).reshape(shape)
    out = v.copy()
    a, b = v[..., :half], v[..., half:rd]
    out[..., :half] = a * c - b * sn
    out[..., half:rd] = a * sn + b * c
    return out


def block_steps(X, p, cache, pos0, s: Shape, kind="tanh", kv_store=None, current_stored=False):
    """``block_step`` for t = 0..T-1 with input X[t] at position pos0 + t, in
    that order (each step appends its K/V and attends over everything
    before it) -- computed with batched projections and one causal softmax
    per row, since the T inputs are known up front (teacher forcing / a
    layer-streamed oracle / prefill).  Equal to the sequential loop up to
    float64 summation order (pinned in tests/test_oracle_golden.py).

    ``kv_store``: as in ``block_step``.  ``current_stored``: the current token
    also attends with its STORED K/V (the batched and prefill device paths read
    it back from the fp16 cache); default False = the fused kernel / the
    sequential ``block_step``."""
    X = np.asarray(X, dtype=np.float64)
    T = X.shape[0]
    if X.ndim != 2 or X.shape[1] != s.hidden:
        raise ValueError(f"inputs must have shape (T, {s.hidden})")
    if len(cache) != pos0:
        raise ValueError(f"cache holds {len(cache)} positions, expected {pos0}")
    H, d = s.n_heads, s.d_head

    def ln_rows(Z, g, b):
        _finite(Z)
        mu = Z.mean(axis=1, keepdims=True)
        var = np.mean((Z - mu) ** 2, axis=1, keepdims=True)
        return (Z - mu) / np.sqrt(var + s.ln_eps) * g + b

    n1 = ln_rows(X, p["ln1_gain"], p["ln1_bias"])
    Y = (n1 @ p["qkv_weight"].T + p["qkv_bias"]).reshape(T, H, 3 * d)
    pos = pos0 + np.arange(T)
    q = rope_rows(Y[:, :, :d], pos, s.rotary_dims, s.theta_base)
    k = rope_rows(Y[:, :, d:2 * d], pos, s.rotary_dims, s.theta_base)
    v = Y[:, :, 2 * d:].copy()
    ks = kv_store(k) if kv_store else k
    vs = kv_store(v) if kv_store else v
    for t in range(T):
        cache.append(ks[t], vs[t])
    Kall = cache.k[:, :pos0 + T].copy()
    Vall = cache.v[:, :pos0 + T].copy()
    scale = 1.0 / math.sqrt(d)
    Qh = q.transpose(1, 0, 2)  # [H, T, d]
    if kv_store and not current_stored:
        # the diagonal (row t, key pos0 + t) uses the exact K/V
        S = np.einsum("htd,hpd->htp", Qh, Kall) * scale
        diag = np.einsum("htd,htd->ht", Qh, k.transpose(1, 0, 2)) * scale
        idx = pos0 + np.arange(T)
        S[:, np.arange(T), idx] = diag
        P = Kall.shape[1]
        mask = np.arange(P)[None, :] > idx[:, None]
        S = np.where(mask[None], -np.inf, S)
        m = S.max(axis=2, keepdims=True)
        w = np.exp(S - m)
        o = np.einsum("htp,hpd->htd", w, Vall)
        wd = w[:, np.arange(T), idx]  # [H, T]
        o += wd[:, :, None] * (v.transpose(1, 0, 2) - vs.transpose(1, 0, 2))
        ctx = o / w.sum(axis=2, keepdims=True)
    else:
        ctx = causal_attention(Qh, Kall, Vall, scale)
    ctx = ctx.transpose(1, 0, 2).reshape(T, s.hidden)
    attn_res = X + ctx @ p["out_weight"].T + p["out_bias"]
    ln2_in = X if s.parallel_residual else attn_res
    n2 = ln_rows(ln2_in, p["ln2_gain"], p["ln2_bias"])
    hdn = n2 @ p["up_weight"].T + p["up_bias"]
    return attn_res + gelu(hdn, kind) @ p["down_weight"].T + p["down_bias"]


def partition_kv(n, blocks):
    """Balanced contiguous ranges, first n % blocks get +1 (nf/cluster.py:134-150)."""
    base, extra = divmod(n, blocks)
    out, a = [], 0
    for b in range(blocks):
        sz = base + (1 if b < extra else 0)
        out.append((a, a + sz))
        a += sz
    return out


def split_attend(q, keys, values, blocks, scale):
    """Split-KV attention with the order-free closed-form merge of EXACT mode
    (nf/cluster.py:172-181, 204-242)."""
    states = [sm_state(q, keys[a:b], values[a:b], scale)
              for a, b in partition_kv(np.asarray(keys).shape[0], blocks)]
    live = [st for st in states if st[1] > 0.0]
    if not live:
        raise ValueError("attention over empty cache")
    m = max(st[0] for st in live)
    f = [math.exp(st[0] - m) for st in live]
    l = math.fsum(st[1] * fi for st, fi in zip(live, f))
    o = np.sum([st[2] * fi for st, fi in zip(live, f)], axis=0)
    return o / l


# ---------------------------------------------------------------------------
# Model-level composition (multi-layer decode + head).

def greedy(logits):
    """argmax, ties toward the lowest index (nf/fidelity.py:27-34)."""
    return int(np.argmax(np.asarray(logits)))


class Model:
    """Layers composed with per-layer seeds; embedding -> blocks -> final LN
    -> unembed.  ``probe=True`` reproduces DecodeInstance's probe head
    (logits = unembed @ h, no final LN: nf/fidelity.py:131-140)."""

    def __init__(self, s: Shape, layers: list, head: dict | None, kind="tanh"):
        self.s, self.layers, self.head, self.kind = s, layers, head, kind
        self.caches = [KV(s.n_heads, s.d_head) for _ in layers]

    def load_prefix(self, keys_per_layer, values_per_layer):
        self.caches = [KV.of(k, v) for k, v in zip(keys_per_layer, values_per_layer)]

    @property
    def pos(self):
        return len(self.caches[0])

    def hidden_states(self, x0, kv_store=None):
        """Returns [x_0, x_1, ..., x_L] for one step (appends to every cache)."""
        xs = [np.asarray(x0, dtype=np.float64)]
        pos = self.pos
        for p, c in zip(self.layers, self.caches):
            xs.append(block_step(xs[-1], p, c, pos, self.s, self.kind, kv_store=kv_store))
        return xs

    def hidden_states_batched(self, X, kv_store=None, current_stored=False):
        """T consecutive tokens with known inputs X [T, h] through all layers
        (``block_steps`` per layer): returns [L+1, T, h]."""
        out = [np.asarray(X, dtype=np.float64)]
        pos = self.pos
        for p, c in zip(self.layers, self.caches):
            out.append(block_steps(out[-1], p, c, pos, self.s, self.kind, kv_store, current_stored))
        return np.array(out)

    def logits(self, h, probe=False):
        hd = self.head
        if not probe:
            h = ln_two_pass(h, hd["lnf_gain"], hd["lnf_bias"], self.s.ln_eps)
        return hd["unembed"] @ h

    def logits_rows(self, H, probe=False):
        """``logits`` of every row of H [T, h]."""
        H = np.asarray(H, np.float64)
        if not probe:
            mu = H.mean(axis=1, keepdims=True)
            var = np.mean((H - mu) ** 2, axis=1, keepdims=True)
            H = (H - mu) / np.sqrt(var + self.s.ln_eps) * self.head["lnf_gain"] + self.head["lnf_bias"]
        return H @ self.head["unembed"].T

    def step_token(self, token, kv_store=None):
        xs = self.hidden_states(self.head["embed"][token], kv_store)
        lg = self.logits(xs[-1])
        return greedy(lg), lg, xs


# ---------------------------------------------------------------------------
# Synthetic KV prefix recipe, as generated on the
# device by nfb_kv_synth: 0.8660254037844386 * u (variance 0.25, the
# reference's N(0,1)*0.5 scale -- nf/fidelity.py:168-169), rounded to fp16.

def kv_seed(base: int, layer: int) -> int:
    return (base + 0x10000 + layer) & _MASK64


def synth_kv(s: Shape, count: int, seed: int):
    n = s.n_heads * count * s.d_head
    k = f16_round(0.8660254037844386 * uniform_stream(seed, 0, n)).reshape(s.n_heads, count, s.d_head)
    v = f16_round(0.8660254037844386 * uniform_stream(seed, 1, n)).reshape(s.n_heads, count, s.d_head)
    return k, v


# ---------------------------------------------------------------------------
# Fast synthesis for the multi-layer tests: oracle/synth.c (the same recipe,
# restated in C; built in-tree by __graft_entry__.build() as
# oracle/liboracle_synth.so; pinned bit-exact against synth_block /
# synth_head / synth_kv by tests/test_oracle_golden.py).  Falls back to numpy.

_CSYNTH = None


def _csynth():
    global _CSYNTH
    if _CSYNTH is None:
        import ctypes
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle_synth.so")
        try:
            lib = ctypes.CDLL(path)
            lib.oracle_synth_f16.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                                             ctypes.c_double, ctypes.c_void_p]
            lib.oracle_synth_f16.restype = None
            lib.oracle_synth_f16_range.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64,
                                                   ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
            lib.oracle_synth_f16_range.restype = None
            _CSYNTH = lib
        except OSError:
            _CSYNTH = False
    return _CSYNTH


def _synth_f16(seed, stream, shape, kind, div=1.0, start=0):
    n = int(np.prod(shape))
    lib = _csynth()
    if not lib:
        u = uniform_stream(seed, stream, start + n)[start:]
        v = {0: u / div, 1: 1.0 + 0.1 * u, 2: 0.1 * u, 3: 0.02 * u, 4: u, 5: 0.8660254037844386 * u}[kind]
        return f16_round(v).reshape(shape)
    out = np.empty(n, np.float64)
    lib.oracle_synth_f16_range(seed & _MASK64, stream, start, n, kind, float(div), out.ctypes.data)
    return out.reshape(shape)


def synth_block_f16(s: Shape, seed: int) -> dict:
    """== f16_params(synth_block(s, seed))."""
    out = {}
    for stream, name in enumerate(BLOCK_TENSORS):
        shape = block_shapes(s)[name]
        if name.endswith("_weight"):
            out[name] = _synth_f16(seed, stream, shape, 0, math.sqrt(shape[1]))
        elif name.endswith("gain"):
            out[name] = _synth_f16(seed, stream, shape, 1)
        elif name in ("ln1_bias", "ln2_bias"):
            out[name] = _synth_f16(seed, stream, shape, 2)
        else:
            out[name] = _synth_f16(seed, stream, shape, 3)
    return out


def synth_head_f16(s: Shape, seed: int) -> dict:
    """== f16_params(synth_head(s, seed))."""
    h, V = s.hidden, s.vocab
    return {"embed": _synth_f16(seed, 0, (V, h), 4), "lnf_gain": _synth_f16(seed, 1, (h,), 1),
            "lnf_bias": _synth_f16(seed, 2, (h,), 2), "unembed": _synth_f16(seed, 3, (V, h), 0, math.sqrt(h))}


def synth_kv_fast(s: Shape, count: int, seed: int, head0: int = 0, n_heads: int | None = None):
    """== synth_kv(s, count, seed) (heads [head0, head0 + n_heads) of a
    stream that may hold more heads, e.g. the batched path's bmax * H)."""
    nh = s.n_heads if n_heads is None else n_heads
    shape = (nh, count, s.d_head)
    a = head0 * count * s.d_head
    return _synth_f16(seed, 0, shape, 5, start=a), _synth_f16(seed, 1, shape, 5, start=a)
