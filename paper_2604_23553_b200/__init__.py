"""B200-native fused GPT-NeoX / Pythia decode block.

Drop-in for the hot path of the reference package ``neoxfuse`` (arXiv
2604.23553, ClusterFusion++): the single-token decode step of a decoder block
runs as one hand-written sm_100a kernel (``libnfb200.so``, C-ABI in
``include/nfb200.h``), behind the reference's Python API.
"""

from .cluster import (
    RING, TREE, ClusterSpec, ExecTrace, KernelTraceRecord, Precision, ReductionKind,
    ReductionStrategy, attend_split, build_trace, fused_block_step, invalidate_weights, output_project_atomic,
    partition_kv,
    release_device_state,
    ring_steps, trace_to_jsonl, tree_steps,
)
from .config import PRESETS, ModelConfig, preset
from .engine import Engine, kv_seed
from .golden import decoder_block_golden, prefill_attention_tiled
from .fidelity import (
    ADVERSARIAL_N_BLOCKS, DecodeInstance, FidelityReport, SweepSummary, adversarial_instance,
    compare, distinct_greedy_outputs, format_report, greedy_tokens, seed_sweep, synthetic_instance, topk_indices,
)
from .perf import (
    ParamCounts, TrafficReport, count_params, flops_per_token, lm_head_bytes, mean_step_bytes,
    step_bytes, traffic,
)
from .plans import (
    NAMED_PLANS, PIPELINE, FusionPlan, Kernel, Op, boundary_tensors, kernel_layer_bytes,
    plan_attention_only, plan_baseline, plan_from_splits, plan_full_fused, plan_mlp_down_only,
)
from .weights import (
    TENSOR_NAMES, BlockWeights, KVCache, load_weights, save_weights, synth_weights,
    to_half_precision,
)

__version__ = "0.1.0"
