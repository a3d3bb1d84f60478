"""CPU-only checks of the host side: byte model (roofline numerator) against
the reference's own numbers, the drop-in Python API surface, and the C-ABI
library (loads and exports every symbol include/nfb200.h declares -- no
compute calls, there is no GPU here)."""

import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_2604_23553_b200 as pkg
from paper_2604_23553_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")


def _bytes_doc():
    with open(os.path.join(G, "bytes.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["pythia-2.8b", "pythia-6.9b", "c1"])
def test_byte_model_matches_reference(name):
    """traffic()/kernel_layer_bytes() integers equal the reference's
    (nf/perfmodel.py:101-121, nf/plans.py:182-211), fixtures from make_golden.py."""
    doc = _bytes_doc()
    cfg = pkg.preset("pythia-160m-shape").with_(n_layers=1) if name == "c1" else pkg.preset(name)
    for P in (1, 129, 1025, 1152, 2049, 4097):
        t = pkg.traffic(pkg.plan_full_fused(), cfg, P)
        assert [t.layer_bytes, t.lm_head_bytes, t.step_bytes] == doc[f"{name}.full.{P}"]
        assert pkg.kernel_layer_bytes(pkg.plan_baseline(), cfg, P) == doc[f"{name}.baseline.{P}"]
    c = pkg.count_params(cfg)
    assert [c.per_layer, c.blocks, c.final_ln, c.unembedding] == doc[f"{name}.params"]
    assert pkg.flops_per_token(cfg, 1024) == doc[f"{name}.flops.1024"]


def test_roofline_numerator_c2():
    """SURVEY.md key numbers: C2 mean bytes over positions 1024..1151."""
    cfg = pkg.preset("pythia-2.8b")
    assert pkg.step_bytes(cfg, 1025) == 5_629_716_480
    assert pkg.mean_step_bytes(cfg, 1024, 128) == 5_650_524_160


def test_partition_kv_rule():
    """First seq % n blocks get one extra position (nf/cluster.py:134-150);
    the kernel's per-rank KV split (csrc/nfb_decode.cu Producer::run) uses
    base = pos / C, extra = pos % C, start = r*base + min(r, extra)."""
    for n in range(0, 40):
        for C in range(1, 9):
            got = pkg.partition_kv(n, C)
            base, extra = divmod(n, C)
            dev = [(r * base + min(r, extra), r * base + min(r, extra) + base + (r < extra))
                   for r in range(C)]
            assert got == dev
            assert got[0][0] == 0 and got[-1][1] == n


def test_model_config_validation_messages():
    with pytest.raises(ValueError, match=r"hidden \(100\) must equal n_heads \* d_head"):
        pkg.ModelConfig(hidden=100, n_heads=3, d_head=32, n_layers=1, d_mlp=4,
                        rotary_pct=0.25, vocab=8)
    with pytest.raises(ValueError, match="even number"):
        pkg.ModelConfig(hidden=12, n_heads=2, d_head=6, n_layers=1, d_mlp=4,
                        rotary_pct=0.25, vocab=8)
    assert pkg.preset("pythia-2.8b").rotary_dims == 20
    assert pkg.preset("pythia-6.9b").rotary_dims == 32


def test_plan_validation_and_trace_accounting():
    cfg = pkg.preset("pythia-2.8b").with_(n_layers=1)
    plan = pkg.plan_full_fused()
    tr = pkg.build_trace(cfg, pkg.ClusterSpec(4), plan, 1025, 2, pkg.TREE)
    assert tr.kernel_count == 1
    assert tr.bytes_offchip == 167_879_680
    assert tr.sync_steps == 4 and tr.dsmem_exchanges == 6
    with pytest.warns(RuntimeWarning):
        pkg.cluster._resolve_reduction(pkg.TREE, 3)


def _declared_symbols():
    with open(_lib.HEADER) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_]+\**\s+\**(nfb_[a-z_0-9]+)\s*\(", src, re.M)))


def test_header_and_binding_agree():
    decl = _declared_symbols()
    assert len(decl) >= 25
    assert sorted(_lib.SIGNATURES) == decl


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libnfb200.so not built (run __graft_entry__.build())")
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared_symbols():
        assert hasattr(raw, name), name
    lib = _lib.load()
    assert lib.nfb_version() >= 100
    # a refused argument reports through nfb_last_error without touching a GPU
    assert lib.nfb_create(None, 0, 16, 0, 0, None) == _lib.NFB_EINVAL
    assert b"null" in lib.nfb_last_error()


def test_library_is_sm100a_only():
    """The shipped cubin is sm_100a SASS (no PTX to JIT to other archs)."""
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libnfb200.so not built")
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_cpu_fallback_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.load()


def test_product_never_imports_oracle():
    pkgdir = os.path.dirname(pkg.__file__)
    for fn in os.listdir(pkgdir):
        if fn.endswith(".py"):
            with open(os.path.join(pkgdir, fn)) as f:
                src = f.read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), fn


def test_kv_cache_duck_type():
    c = pkg.KVCache(2, 4)
    assert len(c) == 0
    k = np.arange(8.0).reshape(2, 4)
    c.append(k, -k)
    c.append(k + 1, -k - 1)
    assert len(c) == 2
    assert np.array_equal(c.head(1)[0][1], k[1] + 1)


def _owner(g, G, T):
    """CTA owning stream-K unit g (csrc/nfb_umma.cuh u_owner)."""
    return ((g + 1) * G + T - 1) // T - 1


@pytest.mark.parametrize("M,N,K", [(7680, 8, 2560), (2560, 32, 2560), (10240, 128, 2560), (2560, 128, 10240),
                                   (50304, 8, 2560), (300, 17, 72), (128, 256, 64)])
def test_gemm_stream_k_plan(M, N, K):
    """The batched GEMM's host plan (csrc/nfb_umma.cu umma_plan) against a
    restatement: CTA i owns units [i*T/G, (i+1)*T/G) of the tiles x k-blocks
    units, every unit has exactly one owner, a tile's pieces are the owners
    of its units in order (the consumers sum piece slots 0..n-1, uout), and
    no tile has more pieces than the partial-slot count the plan allocates."""
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libnfb200.so not built")
    lib = _lib.load()
    out = (ctypes.c_int * 8)()
    assert lib.nfb_gemm_plan(M, N, K, 148, out) == 0
    G, kb, tiles, max_pieces, stages, su, n_pad, smem = list(out)
    T = tiles * kb
    assert kb == -(-K // 64) and tiles == -(-M // 128) and n_pad == -(-N // 8) * 8
    assert G == min(T, 148 * 3 // 2) and stages >= 2 and su >= 1 and smem <= 227 * 1024
    starts = [i * T // G for i in range(G + 1)]
    owner = [None] * T
    for i in range(G):
        for g in range(starts[i], starts[i + 1]):
            assert owner[g] is None
            owner[g] = i
    assert all(o is not None for o in owner)
    assert all(_owner(g, G, T) == owner[g] for g in range(T))
    worst = 0
    for t in range(tiles):
        pieces = sorted({owner[g] for g in range(t * kb, (t + 1) * kb)})
        assert pieces == list(range(pieces[0], pieces[-1] + 1))  # contiguous owners
        worst = max(worst, len(pieces))
    assert worst == max_pieces
    assert lib.nfb_gemm_plan(M, 0, K, 148, out) < 0


def test_golden_entries_reject_bad_arguments_before_touching_the_gpu():
    """The float64 golden entries (nfb_golden_*, nfb_prefill_attention_tiled)
    validate like the reference (nf/golden.py:80-84, 189-205, 234-255) before
    any device work, so the checks run here without a GPU."""
    cfg = pkg.preset("tiny")
    w = pkg.synth_weights(cfg, 1)
    cache = pkg.KVCache(cfg.n_heads, cfg.d_head)
    x = np.zeros(cfg.hidden)
    with pytest.raises(ValueError, match=r"input must have shape"):
        pkg.decoder_block_golden(x[:-1], w, cache, 0, cfg)
    with pytest.raises(ValueError, match="cache holds 0 positions, expected 3"):
        pkg.decoder_block_golden(x, w, cache, 3, cfg)
    with pytest.raises(ValueError, match="unknown gelu variant"):
        pkg.decoder_block_golden(x, w, cache, 0, cfg, gelu="relu")
    q = np.zeros((5, 8))
    with pytest.raises(ValueError, match="tile must be >= 1"):
        pkg.prefill_attention_tiled(q, q, q, 0)
    with pytest.raises(ValueError, match="must share shape"):
        pkg.prefill_attention_tiled(q, q[:4], q, 2)
    # C-ABI level: an odd rotary width is rejected with the reference's message
    lib = _lib.load()
    desc = _lib.ModelDesc(cfg.hidden, cfg.n_heads, cfg.d_head, 1, cfg.d_mlp, 3, cfg.vocab, 1e-5, 1e4, 1, 0)
    arrs = [np.ascontiguousarray(getattr(w, n), dtype=np.float64) for n in pkg.TENSOR_NAMES]
    ptrs = _lib.BlockWeightPtrs(*[a.ctypes.data for a in arrs])
    out = np.empty(cfg.hidden)
    kn = np.empty((cfg.n_heads, cfg.d_head))
    rc = lib.nfb_golden_block_step(ctypes.byref(desc), ctypes.byref(ptrs), _lib.vptr(x), None, None, 0,
                                   _lib.vptr(out), _lib.vptr(kn), _lib.vptr(kn))
    assert rc == _lib.NFB_EINVAL and b"rotary_dims" in lib.nfb_last_error()
    assert lib.nfb_prefill_attention_tiled(_lib.vptr(q), _lib.vptr(q), _lib.vptr(q), 5, 8, 0, 1, 1.0,
                                           _lib.vptr(q)) == _lib.NFB_EINVAL
