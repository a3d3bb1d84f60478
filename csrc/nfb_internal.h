// Internal types shared by the decode kernel and the host-side context.
// Not part of the C-ABI (see include/nfb200.h for that).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

namespace nfb {

// Weight stages carry at most this many matrix rows.
constexpr int kRows = 8;
// Up biases staged in shared memory per layer (static MLP split).
constexpr int kMaxBias = 512;
// Upper bound on consumer warps (hidden <= 16 * 256 = 4096).
constexpr int kMaxConsumerWarps = 16;

// 8-row blocked layout of a [R][K] matrix (R % 8 == 0, K % 32 == 0): each
// group of 8 consecutive rows is stored [K/32][8][32], so a group keeps the
// byte range it has in row-major order and a warp-wide LDS.128 of one
// 512-byte block is the B operand of two m16n8k16 MMAs.  Layout mode 2 of the
// weight upload / synthesis paths (not used by the batch-1 kernel).
__host__ __device__ inline size_t blk8_index(size_t r, size_t k, size_t K) {
  return (r >> 3) * 8 * K + (k >> 5) * 256 + (r & 7) * 32 + (k & 31);
}

// Per-layer device pointers: the "layer descriptor table" built once per
// context (graph mode re-uses it for every step).
struct LayerW {
  const __half* wqkv;   // [3h][h]  reference layout, rows of head j = [3dj, 3d(j+1))
  const __half* woT;    // [h][h]   W_out^T: row k multiplies context element k
  const __half* wup;    // [m][h]
  const __half* wdT;    // [m][h]   W_down^T: row j multiplies gelu(up)_j
  const float* bqkv;    // [3h]
  const float* bo;      // [h]
  const float* bup;     // [m]
  const float* bd;      // [h]
  const float* ln1g;
  const float* ln1b;
  const float* ln2g;
  const float* ln2b;
  __half* kc;           // [H][max_seq][d]  keys, post-RoPE
  __half* vc;           // [H][max_seq][d]
};

struct HeadW {
  const __half* embed;    // [V][h]
  const float* lnfg;      // [h]
  const float* lnfb;      // [h]
  const __half* unembed;  // [V][h]
};

enum InMode : int { IN_X = 0, IN_TOKEN = 1 };
enum HeadMode : int { HEAD_NONE = 0, HEAD_PROBE = 1, HEAD_LM = 2 };

struct Params {
  // shape
  int h, H, d, m, rd, V, max_seq;
  float eps;
  float scale_log2;     // log2(e) / sqrt(d)
  int parallel;         // GPT-NeoX parallel residual
  int gelu_exact;
  int l0, l1;           // layer range of this launch
  // decomposition
  int C;                // cluster size (CTAs per cluster)
  int n_clusters;
  int ncw;              // consumer warps
  int rows_qkv;         // 3d / C  QKV rows per CTA per head
  int rows_o;           // d / C   W_out^T rows per CTA per head
  int stage_rows;       // matrix rows per weight stage (<= kRows)
  int n_slots;
  int slot_bytes;
  int kv_pos;           // positions per KV stage
  // modes
  int in_mode;
  int head_mode;
  int advance_pos;      // graph/decode mode: pos += 1 after the step
  int dyn_mlp;          // 1: MLP chunks grabbed dynamically (not bitwise reproducible)
  int head_weight_pct;  // static schedule: head-stage bytes weighted by this / 100
  int pf_ahead;         // L2 prefetcher lead over the ring producer (bytes); 0 = off
  int mlp_gap;          // MLP pairs slotted after a head's QKV rows and after its KV share
  int fold_all;         // 1: every CTA stores its own split-K partial (no cluster pre-reduce); fold over all CTAs
  int pair;             // stage pairing (consumers take 2 ring stages per step): 1 MLP, 2 QKV, 4 W_out
  int tp_root;          // 1: the fold adds residual + biases (single GPU, or tensor-parallel rank 0)
  int state_update;     // 1: block 0 advances (pos, step) after the first grid barrier
  int vocab_offset;     // global index of local unembedding row 0 (vocab-parallel LM head)
  int vocab_full;       // embedding rows (= V unless the LM head is vocab-sharded)
  int debug;            // DBG_* bits (measurement only: results are garbage)
  // pointers
  const LayerW* layers;
  HeadW head;
  const float2* rope;   // [max_seq][rd/2] (cos, sin), fp32 from f64 host values
  float* xs;            // [(l1-l0)+1][h] hidden states (xs[0] = block input)
  float* rbuf;          // [h] sequential-residual temp
  float* part;          // [n_clusters][h] cluster partial sums
  float* acc;           // [layers][h] atomic split-K accumulators (acc_mode), all zero between launches
  int acc_mode;         // 1: layer end = red.add.v4.f32 of every CTA's partial + ONE grid barrier
  int acc_prereduce;    // acc_mode: cluster ranks first reduce to rank 0 through DSMEM (half the atomics)
  int* ctr;             // [2][ctr_stride] dynamic chunk counters by step parity
  int ctr_stride;
  unsigned long long* gbar;  // grid barrier arrival counter (monotonic)
  int* state;           // [0] pos, [1] step
  unsigned long long* amax;  // [2] packed (ordered logit, ~index) by step parity
  int* tokens;          // [max_seq] token consumed at each step
  float* logits;        // [V] or null
  int* err;             // device error word
  int assist;           // QKV parts per head computed by CTAs without heads (0: off)
  float* yg;            // [H][3d] assist QKV rows (+ bias)
  unsigned* yflag;      // [H * assist] epoch of the rows in yg (release / acquire)
  unsigned* epoch;      // [1] epoch base: advanced by the launch's layer count, never reset
  unsigned long long* trace;  // optional [grid][trace_stride] globaltimer stamps
  int trace_stride;
};

// Trace slots (per CTA): 0 producer ring-full wait (SM cycles), 1 consumer data wait (cycles)
// (thread 0), 2 kernel start, 3 consumer end, 4 head start, 5 head end,
// then per layer l at 8 + 8*l: 0 layer start, 1 QKV exchanged, 2 context
// ready, 3 END reached, 4 after grid barrier #1, 5 after grid barrier #2,
// 6 first KV stage done, 7 attention state published, 8 partial stored
// (before barrier #1), 9 fold done (before barrier #2).
constexpr int kTraceHeader = 16;  // slots 8..15 spare
constexpr int kTracePerLayer = 12;
// Per-stage log of one layer (lrel = n_layers / 2) at the end of each CTA's
// trace row: consumer thread 0 writes 4 words per stage (clock64 before wait,
// after wait, after release; type | n << 8 | flags << 32), the producer 2 words
// per push (before the empty-slot wait, after issue) from kTraceStageProd on.
constexpr int kTraceStageMax = 64;
constexpr int kTraceStageWords = 4 * kTraceStageMax + 2 * kTraceStageMax;
constexpr int kTraceStageProd = 4 * kTraceStageMax;

// Measurement-only modes (NFB_DEBUG env): stages arrive without data, or
// consumers skip the arithmetic.  Used to split producer- vs consumer-bound time.
constexpr int DBG_NO_COPY = 1;
constexpr int DBG_NO_COMPUTE = 2;

// misc[] word holding the ring producer's issued bytes / 16 (read by the
// L2 prefetcher warp).
constexpr int kMiscCum = 56;

// Shared-memory carve-up, computed identically on host and device.
struct Layout {
  int ring, full, empty, desc, bars, ybuf, attst, ctx, ctx2, gpair, wred, red_in, fold, rope, misc, ubias, lw, total;
};

__host__ __device__ inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Layout make_layout(const Params& p) {
  Layout L;
  int o = 0;
  L.ring = o;   o += p.n_slots * p.slot_bytes;
  o = align_up(o, 16);
  L.full = o;   o += 8 * p.n_slots;
  L.empty = o;  o += 8 * p.n_slots;
  L.desc = o;   o += 16 * p.n_slots;
  L.bars = o;   o += 8 * 4;
  L.ybuf = o;   o += 4 * align_up(3 * p.d, 4);
  L.attst = o;  o += 4 * p.C * p.ncw * align_up(p.d + 2, 4);  // [rank][warp] softmax states
  L.ctx = o;    o += 4 * align_up(p.d, 4);
  L.ctx2 = o;   o += 8 * (align_up(p.d, 4) + 8); // context as (c, c) pairs for FFMA2, + 8 zero pairs
  L.gpair = o;  o += 8 * 32 * p.ncw;           // per warp: gelu(up) of the batch as (g, g) pairs
  L.wred = o;   o += 4 * p.ncw * (align_up(p.rows_qkv, 8) > 4 * kRows ? align_up(p.rows_qkv, 8) : 4 * kRows);
  L.red_in = o; o += 4 * (p.C - 1) * p.h;
  L.fold = o;   o += 4 * 32 * p.ncw;
  L.rope = o;   o += 4 * align_up(p.rd, 4);
  o = align_up(o, 16);
  L.misc = o;   o += 4 * 64;
  L.ubias = o;  o += 4 * kMaxBias;
  L.lw = o;     o += 2 * (int)sizeof(LayerW);
  L.total = align_up(o, 128);
  return L;
}

// Device work buffers of the float64 golden block (csrc/nfb_golden.cu).
struct GoldenBufs {
  const double *ln1g, *ln1b, *wqkv, *bqkv, *wo, *bo, *ln2g, *ln2b, *wup, *bup, *wdown, *bdown;
  double *kc, *vc;                // [H][max_seq][d]
  double *n1, *y, *q, *lg, *ctx;  // scratch
  double *attn, *n2, *act;        // attn_res [h], normed2 [h], gelu(up) [m]
  int* bad;                       // set on a non-finite LayerNorm input
};

}  // namespace nfb
