/*
 * nfb200.h -- C-ABI of the B200-native fused GPT-NeoX decode block.
 *
 * The drop-in boundary for the reference package `neoxfuse`
 * (/root/reference/pkg/src/neoxfuse, "nf/" below).  The reference has no FFI:
 * its boundary is a Python function-level API.  Each entry point names the
 * reference interface it replaces; the Python shim `paper_2604_23553_b200`
 * binds these symbols with ctypes.
 *
 * Conventions: plain pointers and sizes, no torch types.  Every function
 * returns NFB_OK (0) or a negative status; nfb_last_error() returns a
 * thread-local message for the last failure.  Host arrays are row-major in the
 * reference layout.  A context is bound to one device and one CUDA stream and
 * is not thread-safe (one context per decode stream, nf SPEC.md:227).
 */
#ifndef NFB200_H
#define NFB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NFB_OK 0
#define NFB_EINVAL (-1)      /* bad argument (reference: ValueError)            */
#define NFB_ECUDA (-2)       /* CUDA runtime failure                            */
#define NFB_ESTATE (-3)      /* call out of order (weights / KV not loaded)     */
#define NFB_EUNSUPPORTED (-4) /* shape the sm_100a kernel does not support       */
#define NFB_EDEVICE (-5)     /* device-side watchdog fired (hang guard)         */

/* Element types of host arrays handed to the library. */
#define NFB_F64 0
#define NFB_F32 1
#define NFB_F16 2

/* Head modes of nfb_forward. */
#define NFB_HEAD_NONE 0
#define NFB_HEAD_PROBE 1 /* logits = unembed @ h            (nf/fidelity.py:139) */
#define NFB_HEAD_LM 2    /* logits = unembed @ LN_f(h)      (nf/perfmodel.py:96) */

typedef struct nfb_ctx nfb_ctx;

/* Replaces ModelConfig (nf/config.py:11-49); rotary_dims = floor(pct*d_head). */
typedef struct {
  int hidden, n_heads, d_head, n_layers, d_mlp, rotary_dims, vocab;
  double ln_eps, theta_base;
  int parallel_residual; /* nf/config.py:22, default 1 */
  int gelu_exact;        /* 0: tanh (nf/golden.py:164, reference default), 1: erf */
} nfb_model_desc;

/* Replaces BlockWeights (nf/weights.py:24-37): reference shapes [out, in]. */
typedef struct {
  const void *ln1_gain, *ln1_bias, *qkv_weight, *qkv_bias, *out_weight, *out_bias;
  const void *ln2_gain, *ln2_bias, *up_weight, *up_bias, *down_weight, *down_bias;
} nfb_block_weights;

typedef struct {
  int grid;          /* CTAs (one per SM) */
  int cluster_size;  /* CTAs per cluster (DSMEM group) */
  int n_clusters;
  int consumer_warps;
  int stage_rows;
  int n_slots;
  int slot_bytes;
  int kv_stage_pos;
  int smem_bytes;
  int max_seq;
  int sm_count;
} nfb_info;

/* Library version (major*10000 + minor*100 + patch). */
int nfb_version(void);
/* Thread-local text of the last error. */
const char* nfb_last_error(void);

/* Create a context for `desc` on `device` with KV capacity `max_seq` per layer.
 * cluster_size 0 = default (2; 3 when max_seq > 4 hidden / 3); max_clusters 0 = as many as fit co-resident.
 * Replaces constructing ModelConfig + KVCache(n_heads, d_head) (nf/weights.py:135). */
int nfb_create(const nfb_model_desc* desc, int device, int max_seq, int cluster_size,
               int max_clusters, nfb_ctx** out);
int nfb_destroy(nfb_ctx* ctx);
int nfb_get_info(nfb_ctx* ctx, nfb_info* info);

/* Upload one layer's parameters (reference layout, dtype NFB_F64/F32/F16);
 * rounded RNE to binary16 on upload.  Replaces passing `w` to
 * fused_block_step / decoder_block_golden (nf/cluster.py:293, nf/golden.py:191). */
int nfb_set_block_weights(nfb_ctx* ctx, int layer, const nfb_block_weights* w, int dtype);
/* Device-side synth_weights(cfg, seed) (nf/weights.py:65-94), bit-exact, then RNE to fp16. */
int nfb_synth_block_weights(nfb_ctx* ctx, int layer, uint64_t seed);
/* Read back one layer's parameters as float32 in the reference layout
 * (each pointer of `out` is a writable float* of the reference shape). */
int nfb_read_block_weights(nfb_ctx* ctx, int layer, const nfb_block_weights* out);
/* Embedding / final LN / unembedding ([vocab, hidden]); any pointer may be NULL
 * to leave that tensor unset.  Replaces DecodeInstance.unembed (nf/fidelity.py:108). */
int nfb_set_head(nfb_ctx* ctx, const void* embed, const void* lnf_gain, const void* lnf_bias,
                 const void* unembed, int dtype);
/* Device-side synthesis of the head with the documented recipe. */
int nfb_synth_head(nfb_ctx* ctx, uint64_t seed);

/* KV cache rows [n_heads][count][d_head] at positions [start, start+count).
 * Replaces KVCache.from_arrays / keys() / values() (nf/weights.py:144-183). */
int nfb_kv_write(nfb_ctx* ctx, int layer, int start, int count, const void* keys,
                 const void* values, int dtype);
int nfb_kv_read(nfb_ctx* ctx, int layer, int start, int count, float* keys, float* values);
/* Synthetic pre-rotated prefix: 0.8660254 * uniform(-1,1) (variance 0.25) from
 * the counter PRNG. */
int nfb_kv_synth(nfb_ctx* ctx, int layer, int count, uint64_t seed);

/* One decode step of one block at position `pos` (the cache must hold exactly
 * `pos` positions; the new K/V is appended at `pos`).  x_in / x_out are HOST
 * float32 [hidden].  Replaces fused_block_step (nf/cluster.py:291-369). */
int nfb_block_step(nfb_ctx* ctx, int layer, int pos, const float* x_in, float* x_out);

/* All layers (+ optional head) for one position, teacher-forced input vector.
 * x_in HOST [hidden]; hidden_out HOST [(n_layers+1)][hidden] or NULL;
 * logits_out HOST [vocab] or NULL.  Replaces one iteration of
 * DecodeInstance.variant_logits (nf/fidelity.py:142-153). */
int nfb_forward(nfb_ctx* ctx, int pos, const float* x_in, float* hidden_out, float* logits_out,
                int head_mode);

/* Device-resident variants for callers holding torch CUDA tensors (raw
 * pointer + stream; SURVEY.md §8b "Ownership"): x_in / x_out / hidden_out /
 * logits_out are DEVICE float32 pointers, `stream` a cudaStream_t (NULL = the
 * context stream).  Everything is enqueued on `stream` with no host
 * synchronisation (the input is not checked for non-finite values -- that
 * would need a device->host read); a device-side failure surfaces at the next
 * nfb_sync.  Same semantics as nfb_block_step / nfb_forward otherwise. */
int nfb_block_step_dev(nfb_ctx* ctx, int layer, int pos, const float* x_in, float* x_out, void* stream);
int nfb_forward_dev(nfb_ctx* ctx, int pos, const float* x_in, float* hidden_out, float* logits_out,
                    int head_mode, void* stream);

/* Greedy token decode with device-resident state (graph mode).
 * nfb_begin_decode sets position and first input token; each nfb_decode_step
 * embeds the previous argmax, runs all layers + LM head, argmax on device and
 * advances the position.  `stream` may be NULL (context stream). */
int nfb_begin_decode(nfb_ctx* ctx, int pos, int token);
int nfb_decode_step(nfb_ctx* ctx, void* stream);
/* End-to-end serving step with HOST buffers: copy `token` host->device,
 * run one decode step (graph replay if captured, else a launch), copy the
 * argmax device->host into *next_token and wait for it. */
int nfb_step_token(nfb_ctx* ctx, int token, int* next_token);
/* Capture one nfb_decode_step into a CUDA graph; replay it n times. */
int nfb_graph_capture(nfb_ctx* ctx);
int nfb_graph_replay(nfb_ctx* ctx, int n, void* stream);
/* Tokens consumed by steps [0, n) and the argmax of the last step. */
int nfb_read_tokens(nfb_ctx* ctx, int* tokens, int n, int* last_argmax);
/* Hidden states [(n_layers+1)][hidden] and logits [vocab] of the last launch. */
int nfb_read_hidden(nfb_ctx* ctx, float* out);
int nfb_read_logits(nfb_ctx* ctx, float* out);
/* Current device position / step counters. */
int nfb_get_state(nfb_ctx* ctx, int* pos, int* step);
/* Options: NFB_OPT_TRACE (per-CTA globaltimer phase stamps, see
 * csrc/nfb_internal.h), NFB_OPT_DYNAMIC_MLP (work-stealing MLP chunks: not
 * bitwise reproducible), NFB_OPT_PREFETCH_KB.  Invalidates a captured graph. */
#define NFB_OPT_TRACE 1
#define NFB_OPT_DYNAMIC_MLP 2
#define NFB_OPT_PREFETCH_KB 3 /* L2 prefetch lead of the prefetcher warp, KiB (0 = off) */
#define NFB_OPT_HEAD_WEIGHT 4 /* static MLP split: head bytes weighted by value / 100 (default 130) */
#define NFB_OPT_ASSIST 5      /* QKV parts per head computed by CTAs without heads (0 = off) */
#define NFB_OPT_DETERMINISTIC 6 /* 1: fixed-order fold at each layer end (bitwise reproducible run to run);
                                 * 0 (default): fp32 vector atomics + one grid barrier per layer */
int nfb_set_option(nfb_ctx* ctx, int option, int value);
/* Copy up to n trace words ([grid][8 + 12*n_layers]) to `out`. */
int nfb_read_trace(nfb_ctx* ctx, unsigned long long* out, int n);
/* Block until the context stream is idle; reports device-side failures. */
int nfb_sync(nfb_ctx* ctx);

/* ---- tensor parallelism (Pythia-6.9B, BASELINE.json configs[2]) ----------
 * Not in the reference (a single-process simulator): heads, FFN rows and the
 * vocabulary are sharded over tp_size GPUs; each layer is one launch that
 * leaves this rank's split-K partial (rank 0 adds residual + biases) and an
 * NCCL all-reduce sums the ranks -- one per layer thanks to GPT-NeoX's
 * parallel residual (nf/config.py:22, nf/golden.py:224-228).
 * nfb_create_tp takes the FULL model description; the context holds shard
 * tp_rank (weights only via nfb_synth_*; KV I/O addresses the local heads). */
int nfb_create_tp(const nfb_model_desc* full, int device, int max_seq, int cluster_size,
                  int max_clusters, int tp_rank, int tp_size, nfb_ctx** out);
/* NCCL unique id (128 bytes) made on one rank, shared by the caller. */
int nfb_tp_unique_id(void* out128);
/* Join the tp_size-rank NCCL communicator; enables the decode API. */
int nfb_tp_init(nfb_ctx* ctx, const void* unique_id128);
int nfb_tp_info(nfb_ctx* ctx, int* tp_rank, int* tp_size);
/* LM / probe head on a given final hidden state h_in[hidden] -> this
 * context's logits (its vocab shard under TP).  Replaces the probe
 * `unembed @ h` of DecodeInstance (nf/fidelity.py:139, 152). */
int nfb_head_logits(nfb_ctx* ctx, const float* h_in, float* logits_out, int head_mode);

/* ---- batched decode (BASELINE.json configs[3]: batch sweep 1/4/16/64) -------
 * B sequences of one context (its weights) at the same position, each with its
 * own KV cache.  Not in the reference (batch 1 only): the
 * projections run as fp16 GEMMs on hi/lo activation rows (our mma.sync kernel
 * at 2B <= 8 rows, cuBLAS above), attention / RoPE / LN / GELU / residual /
 * argmax in our kernels (csrc/nfb_batch.cu).
 * Parallel residual only. */
int nfb_batch_init(nfb_ctx* ctx, int max_batch);
/* Synthetic prefix of every layer for all max_batch sequences (seed kv_seed(base, l)). */
int nfb_batch_kv_synth(nfb_ctx* ctx, int count, uint64_t base_seed);
int nfb_batch_kv_write(nfb_ctx* ctx, int layer, int seq, int start, int count, const void* keys,
                       const void* values, int dtype);
/* One step of `batch` sequences from inputs x_in[batch][hidden] at `pos` (the
 * K/V of pos are appended); x_out / logits_out (LM head) optional. */
int nfb_batch_forward(nfb_ctx* ctx, int batch, int pos, const float* x_in, float* x_out, float* logits_out);
int nfb_batch_begin(nfb_ctx* ctx, int batch, int pos, const int* tokens);
int nfb_batch_step(nfb_ctx* ctx, int n, void* stream);
int nfb_batch_graph_capture(nfb_ctx* ctx);
int nfb_batch_read_tokens(nfb_ctx* ctx, int* tokens);
/* Prefill (reference prefill_attention_tiled, nf/golden.py:234-265):
 * `count` prompt positions pos.. from inputs x_in[count][hidden] through all
 * layers, causal attention, K/V appended to the context's cache (which must
 * hold exactly `pos` positions), final hidden states to x_out (optional).
 * Runs on the batched kernels in chunks of max_batch rows (nfb_batch_init). */
int nfb_prefill(nfb_ctx* ctx, int pos, int count, const float* x_in, float* x_out);
/* Diagnostics: the batched-projection GEMM (csrc/nfb_umma.cu: tcgen05 + TMEM,
 * weights pre-blocked into the UMMA SW128 layout and streamed with 1-D bulk
 * copies, stream-K partials summed in piece order) on caller-owned DEVICE
 * buffers: Y[N][M] (fp32) = W[M][K] (fp16, row-major) . A[N][K]^T (fp16),
 * N <= 256, enqueued on `stream` (NULL = legacy default).  Not in the
 * reference; used by the unit test / microbenchmark of that kernel.  Return 0
 * or a negative code.  Not thread-safe (one shared workspace).
 *   nfb_gemm_f16_dev          blocks W into the workspace, then runs;
 *   nfb_gemm_blocked_bytes    size of the blocked copy of an M x K matrix;
 *   nfb_gemm_block_weights_dev  W (row-major) -> Wb (blocked), on `stream`;
 *   nfb_gemm_f16_blocked_dev  runs on a pre-blocked Wb (the batched path's
 *                             steady state: weights blocked once). */
int nfb_gemm_f16_dev(int M, int N, int K, const void* W, const void* A, float* Y, void* stream);
size_t nfb_gemm_blocked_bytes(int M, int K);
int nfb_gemm_block_weights_dev(int M, int K, const void* W, void* Wb, void* stream);
int nfb_gemm_f16_blocked_dev(int M, int N, int K, const void* Wb, const void* A, float* Y, void* stream);
/* Diagnostics: per-CTA globaltimer stamps ([grid][8] u64, caller-owned device
 * buffer; NULL turns it off) of the following standalone GEMM launches. */
int nfb_gemm_trace_dev(void* buf);
/* Host-only: the GEMM's stream-K plan for an M x K weight and N activation
 * rows on `sm_count` SMs -> out[8] = {grid, k-blocks per tile, tiles, max
 * pieces per tile, ring stages, units per stage, n_pad, smem bytes}. */
int nfb_gemm_plan(int M, int N, int K, int sm_count, int* out);

/* Unit-level helpers of the reference's cluster simulator, on the GPU
 * (csrc/nfb_split.cu; float64 host arrays, synchronous, current device).
 *
 * nfb_attend_split replaces neoxfuse.cluster.attend_split (nf/cluster.py:211-242):
 * one head, q[d], keys/values[seq_len][d]; the history split into n_blocks
 * ranges by the partition_kv rule (nf/cluster.py:134-150), one softmax state
 * per range, merged in `merge` order: NFB_MERGE_EXACT (closed form,
 * nf/cluster.py:172-181), RING, TREE (power-of-two n_blocks; the caller
 * resolves non-powers to RING with the reference's warning) or PERMUTED
 * (order permutation(n_blocks, seed), nf/halfnum.py:62-74).  out[d].
 *
 * nfb_output_project_atomic replaces neoxfuse.cluster.output_project_atomic
 * (nf/cluster.py:253-285): partials[n_blocks][hidden] projected through
 * w_out[hidden][hidden] and accumulated into residual + b_out; fp16 != 0
 * models FP16 atomic adds (per element j: order permutation(n_blocks,
 * counter_rand_u64(seed, j)), binary16 rounding after every add), else the
 * block contributions are summed in float64.  out[hidden]. */
#define NFB_MERGE_EXACT 0
#define NFB_MERGE_RING 1
#define NFB_MERGE_TREE 2
#define NFB_MERGE_PERMUTED 3
int nfb_attend_split(const double* q, const double* keys, const double* values, int seq_len, int d, int n_blocks,
                     int merge, uint64_t seed, double scale, double* out);
int nfb_output_project_atomic(const double* partials, const double* w_out, const double* b_out,
                              const double* residual, int n_blocks, int hidden, int fp16, uint64_t seed,
                              double* out);

/* nfb_golden_logits replaces neoxfuse.fidelity.DecodeInstance.golden_logits
 * (nf/fidelity.py:131-140): the float64 golden block decoder_block_golden
 * (nf/golden.py:189-228; weights used as given, two-pass LayerNorm, naive
 * per-head softmax over the cache incl. the fresh token) stepped over
 * xs[steps][hidden] from a fresh cache holding prompt_k / prompt_v
 * [n_heads][prompt_len][d_head] (keys already rotated), logits[steps][vocab] =
 * unembed[vocab][hidden] @ h per step.  Model from `m` (n_layers ignored;
 * gelu_exact, parallel_residual, ln_eps, theta_base, rotary_dims used);
 * float64 host arrays, weights in the reference [out, in] shapes; runs on the
 * current device in float64 (csrc/nfb_golden.cu), synchronous.  A non-finite
 * LayerNorm input returns NFB_EINVAL "non-finite activation"
 * (nf/golden.py:29-31). */
int nfb_golden_logits(const nfb_model_desc* m, const nfb_block_weights* w, const double* unembed, const double* xs,
                      int steps, const double* prompt_k, const double* prompt_v, int prompt_len, double* logits);
/* nfb_golden_block_step replaces neoxfuse.golden.decoder_block_golden
 * (nf/golden.py:189-228): one float64 golden step of the block at pos = len
 * over the history keys / values [n_heads][len][d_head] (float64, keys
 * rotated); out[hidden] and the step's rotated key / value k_new, v_new
 * [n_heads][d_head] for the caller's cache append.  Same model fields,
 * device and errors as nfb_golden_logits. */
int nfb_golden_block_step(const nfb_model_desc* m, const nfb_block_weights* w, const double* x, const double* keys,
                          const double* values, int len, double* out, double* k_new, double* v_new);
/* nfb_prefill_attention_tiled replaces neoxfuse.golden.prefill_attention_tiled
 * (nf/golden.py:234-265): one head, Q, K, V [seq][d_head] float64; each query
 * row folds its keys [0, i] (causal != 0) or [0, seq) in tiles of `tile`
 * positions into a running softmax state; out [seq][d_head].  float64 on the
 * current device (csrc/nfb_golden.cu), synchronous. */
int nfb_prefill_attention_tiled(const double* Q, const double* K, const double* V, int seq, int d, int tile,
                                int causal, double scale, double* out);

/* The context's CUDA stream (cudaStream_t) for event timing. */
void* nfb_stream(nfb_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* NFB200_H */
