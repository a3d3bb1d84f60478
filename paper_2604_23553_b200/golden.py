"""The reference's golden block, ``decoder_block_golden`` (nf/golden.py:189-228),
in float64 on the GPU (``nfb_golden_block_step`` / ``nfb_golden_logits``,
csrc/nfb_golden.cu).

The golden block is the unfused float64 pipeline the fused kernel is judged
against; callers of the reference API (``DecodeInstance.golden_logits``,
fidelity sweeps, the reference CLI's golden command) use it next to the fused
path.  Same signature, cache semantics (exactly one appended position, keys
stored rotated) and errors as the reference.  Summation orders differ from
numpy/BLAS, so results agree with the reference to float64 rounding, not
bitwise.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .weights import TENSOR_NAMES


def _desc(cfg, gelu: str):
    if gelu not in ("tanh", "exact"):
        raise ValueError(f"unknown gelu variant {gelu!r} (use 'exact' or 'tanh')")
    return _lib.ModelDesc(cfg.hidden, cfg.n_heads, cfg.d_head, 1, cfg.d_mlp, cfg.rotary_dims, cfg.vocab,
                          float(cfg.ln_eps), float(cfg.theta_base), 1 if cfg.parallel_residual else 0,
                          1 if gelu == "exact" else 0)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _weight_ptrs(w):
    """(BlockWeightPtrs, the float64 arrays they point into -- keep alive)."""
    arrs = [_f64(getattr(w, n)) for n in TENSOR_NAMES]
    return _lib.BlockWeightPtrs(*[a.ctypes.data for a in arrs]), arrs


def decoder_block_golden(x, w, cache, pos: int, cfg, gelu: str = "tanh") -> np.ndarray:
    """One decode step of the unfused block in float64 (nf/golden.py:189-228):
    parallel residual ``x + attention(ln1(x)) + mlp(ln2(x))``, or sequential
    ``r = x + attention(ln1(x)); r + mlp(ln2(r))``; appends this step's K/V
    to ``cache``, which must hold exactly the positions < pos."""
    x = _f64(x)
    if x.shape != (cfg.hidden,):
        raise ValueError(f"input must have shape ({cfg.hidden},)")
    if len(cache) != pos:
        raise ValueError(f"cache holds {len(cache)} positions, expected {pos}")
    desc = _desc(cfg, gelu)
    w.validate(cfg)
    ptrs, keep = _weight_ptrs(w)
    keys, values = _f64(cache.keys()), _f64(cache.values())
    out = np.empty(cfg.hidden)
    k_new = np.empty((cfg.n_heads, cfg.d_head))
    v_new = np.empty((cfg.n_heads, cfg.d_head))
    lib = _lib.load()
    _lib.check(lib.nfb_golden_block_step(C.byref(desc), C.byref(ptrs), _lib.vptr(x), _lib.vptr(keys),
                                         _lib.vptr(values), int(pos), _lib.vptr(out), _lib.vptr(k_new),
                                         _lib.vptr(v_new)), "decoder_block_golden")
    del keep
    cache.append(k_new, v_new)
    return out


def golden_logits(cfg, w, unembed, xs, prompt_keys, prompt_values, gelu: str = "tanh") -> np.ndarray:
    """``decoder_block_golden`` stepped over ``xs`` from a fresh cache holding
    the prompt K/V, ``unembed @ h`` per step (nf/fidelity.py:131-140)."""
    desc = _desc(cfg, gelu)
    ptrs, keep = _weight_ptrs(w)
    un, xs = _f64(unembed), _f64(xs)
    pk, pv = _f64(prompt_keys), _f64(prompt_values)
    out = np.empty((xs.shape[0], cfg.vocab))
    lib = _lib.load()
    _lib.check(lib.nfb_golden_logits(C.byref(desc), C.byref(ptrs), _lib.vptr(un), _lib.vptr(xs), xs.shape[0],
                                     _lib.vptr(pk), _lib.vptr(pv), pk.shape[1], _lib.vptr(out)), "golden_logits")
    del keep
    return out


def prefill_attention_tiled(Q, K, V, tile: int, causal: bool = True, scale: float | None = None) -> np.ndarray:
    """Causal (or full) attention of one head over whole sequences, keys folded
    in tiles of ``tile`` positions into a running softmax state per query row
    (nf/golden.py:234-265), in float64 on the GPU
    (``nfb_prefill_attention_tiled``).  Q, K, V: [seq, d_head]."""
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    if Q.ndim != 2 or K.shape != Q.shape or V.shape != Q.shape:
        raise ValueError("Q, K, V must share shape [seq, d_head]")
    if tile < 1:
        raise ValueError("tile must be >= 1")
    seq, d = Q.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    out = np.empty((seq, d))
    if seq == 0:
        return out
    lib = _lib.load()
    _lib.check(lib.nfb_prefill_attention_tiled(_lib.vptr(Q), _lib.vptr(K), _lib.vptr(V), seq, d, int(tile),
                                               1 if causal else 0, float(scale), _lib.vptr(out)),
               "prefill_attention_tiled")
    return out
