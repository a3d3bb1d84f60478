"""ctypes binding of the C-ABI library ``libnfb200.so`` (include/nfb200.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no CPU
fallback: if the library (or a GPU) is missing, every compute call raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# NFB_LIB: load another build of the library (A/B measurements in tools/)
LIB_PATH = os.environ.get("NFB_LIB") or os.path.join(_HERE, "libnfb200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "nfb200.h")

NFB_OK, NFB_EINVAL, NFB_ECUDA, NFB_ESTATE, NFB_EUNSUPPORTED, NFB_EDEVICE = 0, -1, -2, -3, -4, -5
NFB_F64, NFB_F32, NFB_F16 = 0, 1, 2
MERGE_EXACT, MERGE_RING, MERGE_TREE, MERGE_PERMUTED = 0, 1, 2, 3
HEAD_NONE, HEAD_PROBE, HEAD_LM = 0, 1, 2
OPT_TRACE, OPT_DYNAMIC_MLP, OPT_PREFETCH_KB, OPT_HEAD_WEIGHT, OPT_ASSIST, OPT_DETERMINISTIC = 1, 2, 3, 4, 5, 6


class ModelDesc(C.Structure):
    _fields_ = [
        ("hidden", C.c_int), ("n_heads", C.c_int), ("d_head", C.c_int), ("n_layers", C.c_int),
        ("d_mlp", C.c_int), ("rotary_dims", C.c_int), ("vocab", C.c_int),
        ("ln_eps", C.c_double), ("theta_base", C.c_double),
        ("parallel_residual", C.c_int), ("gelu_exact", C.c_int),
    ]


class BlockWeightPtrs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "ln1_gain", "ln1_bias", "qkv_weight", "qkv_bias", "out_weight", "out_bias",
        "ln2_gain", "ln2_bias", "up_weight", "up_bias", "down_weight", "down_bias")]


class Info(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "grid", "cluster_size", "n_clusters", "consumer_warps", "stage_rows", "n_slots",
        "slot_bytes", "kv_stage_pos", "smem_bytes", "max_seq", "sm_count")]


class UnsupportedShapeError(ValueError):
    """The sm_100a kernel does not support this model shape."""


_P = C.c_void_p
_I = C.c_int
_FP = C.POINTER(C.c_float)
_IP = C.POINTER(C.c_int)

# name -> (restype, argtypes); every symbol declared in include/nfb200.h
SIGNATURES = {
    "nfb_version": (_I, []),
    "nfb_last_error": (C.c_char_p, []),
    "nfb_create": (_I, [C.POINTER(ModelDesc), _I, _I, _I, _I, C.POINTER(_P)]),
    "nfb_destroy": (_I, [_P]),
    "nfb_get_info": (_I, [_P, C.POINTER(Info)]),
    "nfb_set_block_weights": (_I, [_P, _I, C.POINTER(BlockWeightPtrs), _I]),
    "nfb_synth_block_weights": (_I, [_P, _I, C.c_uint64]),
    "nfb_read_block_weights": (_I, [_P, _I, C.POINTER(BlockWeightPtrs)]),
    "nfb_set_head": (_I, [_P, _P, _P, _P, _P, _I]),
    "nfb_synth_head": (_I, [_P, C.c_uint64]),
    "nfb_kv_write": (_I, [_P, _I, _I, _I, _P, _P, _I]),
    "nfb_kv_read": (_I, [_P, _I, _I, _I, _FP, _FP]),
    "nfb_kv_synth": (_I, [_P, _I, _I, C.c_uint64]),
    "nfb_block_step": (_I, [_P, _I, _I, _FP, _FP]),
    "nfb_forward": (_I, [_P, _I, _FP, _FP, _FP, _I]),
    "nfb_block_step_dev": (_I, [_P, _I, _I, _P, _P, _P]),
    "nfb_gemm_f16_dev": (_I, [_I, _I, _I, _P, _P, _P, _P]),
    "nfb_gemm_blocked_bytes": (C.c_size_t, [_I, _I]),
    "nfb_gemm_block_weights_dev": (_I, [_I, _I, _P, _P, _P]),
    "nfb_gemm_f16_blocked_dev": (_I, [_I, _I, _I, _P, _P, _P, _P]),
    "nfb_gemm_trace_dev": (_I, [_P]),
    "nfb_gemm_plan": (_I, [_I, _I, _I, _I, _IP]),
    "nfb_forward_dev": (_I, [_P, _I, _P, _P, _P, _I, _P]),
    "nfb_begin_decode": (_I, [_P, _I, _I]),
    "nfb_decode_step": (_I, [_P, _P]),
    "nfb_step_token": (_I, [_P, _I, _IP]),
    "nfb_graph_capture": (_I, [_P]),
    "nfb_graph_replay": (_I, [_P, _I, _P]),
    "nfb_read_tokens": (_I, [_P, _IP, _I, _IP]),
    "nfb_read_hidden": (_I, [_P, _FP]),
    "nfb_read_logits": (_I, [_P, _FP]),
    "nfb_get_state": (_I, [_P, _IP, _IP]),
    "nfb_sync": (_I, [_P]),
    "nfb_set_option": (_I, [_P, _I, _I]),
    "nfb_read_trace": (_I, [_P, C.POINTER(C.c_ulonglong), _I]),
    "nfb_stream": (_P, [_P]),
    "nfb_create_tp": (_I, [C.POINTER(ModelDesc), _I, _I, _I, _I, _I, _I, C.POINTER(_P)]),
    "nfb_tp_unique_id": (_I, [_P]),
    "nfb_tp_init": (_I, [_P, _P]),
    "nfb_tp_info": (_I, [_P, _IP, _IP]),
    "nfb_head_logits": (_I, [_P, _FP, _FP, _I]),
    "nfb_batch_init": (_I, [_P, _I]),
    "nfb_batch_kv_synth": (_I, [_P, _I, C.c_uint64]),
    "nfb_batch_kv_write": (_I, [_P, _I, _I, _I, _I, _P, _P, _I]),
    "nfb_batch_forward": (_I, [_P, _I, _I, _FP, _FP, _FP]),
    "nfb_batch_begin": (_I, [_P, _I, _I, _IP]),
    "nfb_batch_step": (_I, [_P, _I, _P]),
    "nfb_batch_graph_capture": (_I, [_P]),
    "nfb_batch_read_tokens": (_I, [_P, _IP]),
    "nfb_prefill": (_I, [_P, _I, _I, _FP, _FP]),
    "nfb_attend_split": (_I, [_P, _P, _P, _I, _I, _I, _I, C.c_uint64, C.c_double, _P]),
    "nfb_output_project_atomic": (_I, [_P, _P, _P, _P, _I, _I, _I, C.c_uint64, _P]),
    "nfb_golden_logits": (_I, [C.POINTER(ModelDesc), C.POINTER(BlockWeightPtrs), _P, _P, _I, _P, _P, _I, _P]),
    "nfb_golden_block_step": (_I, [C.POINTER(ModelDesc), C.POINTER(BlockWeightPtrs), _P, _P, _P, _I, _P, _P, _P]),
    "nfb_prefill_attention_tiled": (_I, [_P, _P, _P, _I, _I, _I, _I, C.c_double, _P]),
}

_lib = None


def _prefer_torch_nccl() -> None:
    """Point the library's lazy NCCL dlopen at the NCCL torch bundles (the
    nvidia-nccl wheel), found without importing torch: if the system
    libnccl.so.2 were loaded first, a later `import torch` would resolve its
    libnccl.so.2 dependency to that older library and fail."""
    if os.environ.get("NFB_NCCL_LIB"):
        return
    import importlib.util
    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for d in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["NFB_NCCL_LIB"] = cand
            return


def load():
    """Load the in-tree library; raises ImportError (no fallback) if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the fused decode block has no CPU fallback)")
    _prefer_torch_nccl()
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    if status == NFB_OK:
        return
    msg = load().nfb_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == NFB_EINVAL:
        raise ValueError(msg)
    if status == NFB_EUNSUPPORTED:
        raise UnsupportedShapeError(msg)
    raise RuntimeError(f"[nfb status {status}] {msg}")


def fptr(a):
    return a.ctypes.data_as(_FP)


def vptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None
