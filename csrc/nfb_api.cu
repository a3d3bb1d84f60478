// C-ABI implementation (include/nfb200.h): context, parameter upload and
// device-side synthesis, KV cache I/O, launch paths (eager, decode, graph).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../include/nfb200.h"
#include "nfb_internal.h"
#include "nfb_umma.cuh"

namespace nfb {
const void* decode_kernel_ptr(int dpl);
// batched decode kernels (csrc/nfb_batch.cu)
__global__ void ln_hilo_kernel(const float* x, int B, int h, float eps, const float* g1, const float* b1,
                               const float* g2, const float* b2, __half* a1, __half* a2, int n_pad);
__global__ void attn_prep_kernel(const UOut y, int B, int H, int d, int rd, const int* state, int max_seq,
                                 const float* bqkv, const float2* rope, float* q, __half* kc, __half* vc,
                                 int pos_step, size_t seq_stride);
__global__ void attn_combine_kernel(const float* part, int S, int B, int H, int d, __half* ctx, int n_pad);
__global__ void attn_tile_kernel(const float* q, const __half* kc, const __half* vc, int B, int H, int d,
                                 int max_seq, const int* state, float scale_log2, float* part, int pos_step,
                                 size_t seq_stride);
size_t attn_tile_smem(int d);
int attn_tile_positions();
int attn_prefill_rows();
size_t attn_tile_rows_smem(int d);
__global__ void attn_tile_rows_kernel(const float* q, const __half* kc, const __half* vc, int T, int H, int d,
                                      int max_seq, const int* state, float scale_log2, float* part);
// tcgen05 GEMM (csrc/nfb_umma.cu)
UPlan umma_plan(int M, int N, int K, int sm_count);
size_t umma_blocked_elems(int M, int K);
size_t umma_act_elems(int n_pad, int K);
UOut umma_out(const UPlan& P, const float* ws);
void umma_block_weights(cudaStream_t st, const __half* src, int M, int K, size_t ld, bool trans, __half* dst);
cudaError_t umma_gemm(cudaStream_t st, const UPlan& P, const void* Wb, const void* Ab, float* ws, int* err, bool pdl,
                      unsigned long long* trace = nullptr);
__global__ void gelu_hilo_kernel(const UOut u, int B, int m, const float* bup, int exact, __half* g, int n_pad);
__global__ void residual_kernel(float* x, int B, int h, const UOut z, const float* bo, const UOut dn,
                                const float* bd);
__global__ void argmax_kernel(const UOut lg, int B, int V, unsigned long long* amax, float* logits_out);
__global__ void embed_kernel(const int* tokens, const __half* embed, int h, int V, float* x);
__global__ void advance_kernel(int* state, unsigned long long* amax, int* tokens, int B, int V);
cudaError_t launch_decode(const Params& p, int dpl, int grid, int block, int smem, cudaStream_t st,
                          bool cooperative);
cudaError_t max_active_clusters(int dpl, int C, int block, int smem, int* out);
// single-head split-KV attention / atomic output projection (csrc/nfb_split.cu)
cudaError_t golden_step(const GoldenBufs& B, const double* x, double* out, int h, int H, int d, int m, int rd,
                        double eps, double base, int pos, int max_seq, int parallel, int gelu_exact,
                        cudaStream_t st);
cudaError_t golden_probe(const double* unembed, const double* hv, int vocab, int h, double* logits, cudaStream_t st);
cudaError_t golden_prefill_tiled(const double* Q, const double* K, const double* V, int seq, int d, int tile,
                                 int causal, double scale, double* out, cudaStream_t st);
cudaError_t launch_attend_split(const double* q, const double* K, const double* V, int seq, int d, int n, int mode,
                                uint64_t seed, double scale, double* logits, double* states, int* order,
                                void* scratch, double* out, cudaStream_t st);
size_t attend_split_scratch_bytes(int n, int d);
cudaError_t launch_project_atomic(const double* P, const double* W, const double* bias, const double* residual,
                                  int n, int hidden, int fp16, uint64_t seed, double* proj, int* order, double* out,
                                  cudaStream_t st);
}  // namespace nfb

using namespace nfb;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(expr)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(NFB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));     \
  } while (0)

// ---------------------------------------------------------------------------
// NCCL, loaded on first use (the library links no NCCL: single-GPU users need
// none, and under torch the already-loaded libnccl.so.2 is reused).
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

static NcclApi& nccl_api() {
  static NcclApi a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // NFB_NCCL_LIB (set by the Python shim to the NCCL that torch bundles):
    // loading the system libnccl.so.2 first would make a later `import torch`
    // bind its libnccl.so.2 dependency to that older library
    void* h = nullptr;
    if (const char* path = getenv("NFB_NCCL_LIB")) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
      a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
      a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
      a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
      a.getErrorString = (decltype(a.getErrorString))dlsym(h, "ncclGetErrorString");
      a.ok = a.getUniqueId && a.commInitRank && a.allReduce && a.commDestroy && a.getErrorString;
    }
  }
  return a;
}

#define NCK(expr)                                                                          \
  do {                                                                                     \
    ncclResult_t r_ = (expr);                                                              \
    if (r_ != ncclSuccess) return fail(NFB_ECUDA, std::string(#expr) + ": " + nccl_api().getErrorString(r_)); \
  } while (0)



// ---------------------------------------------------------------------------
// binary16 round-to-nearest-even from float64 bits (IEEE 754; same results as
// the reference's integer algorithm, nf/halfnum.py:80-111).
__host__ __device__ inline uint16_t f64_to_f16_bits(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  const uint16_t sign = (uint16_t)((b >> 48) & 0x8000u);
  const int ex = (int)((b >> 52) & 0x7ff);
  const uint64_t frac = b & 0xfffffffffffffull;
  if (ex == 0x7ff) return frac ? 0x7e00 : (uint16_t)(sign | 0x7c00);
  const int e = ex - 1023;
  if (e >= 16) return (uint16_t)(sign | 0x7c00);
  if (e >= -14) {
    uint32_t hv = ((uint32_t)(e + 15) << 10) | (uint32_t)(frac >> 42);
    const uint64_t rest = frac & ((1ull << 42) - 1);
    const uint64_t tie = 1ull << 41;
    if (rest > tie || (rest == tie && (hv & 1u))) ++hv;
    return (uint16_t)(sign | hv);
  }
  if (e < -26) return sign;
  const uint64_t sig = (1ull << 52) | frac;
  const int sh = 28 - e;
  uint64_t q = sig >> sh;
  const uint64_t rest = sig & ((1ull << sh) - 1);
  const uint64_t tie = 1ull << (sh - 1);
  if (rest > tie || (rest == tie && (q & 1ull))) ++q;
  return (uint16_t)(sign | q);
}

__host__ __device__ inline float f16_bits_to_f32(uint16_t hb) {
  const uint32_t sign = (uint32_t)(hb & 0x8000u) << 16;
  const uint32_t ex = (hb >> 10) & 0x1f, fr = hb & 0x3ffu;
  float v;
  if (ex == 0) {
    v = (float)fr * 5.9604644775390625e-08f;  // 2^-24
    uint32_t u;
    memcpy(&u, &v, 4);
    u |= sign;
    memcpy(&v, &u, 4);
    return v;
  }
  uint32_t u = ex == 31 ? (sign | 0x7f800000u | (fr << 13)) : (sign | ((ex + 112) << 23) | (fr << 13));
  memcpy(&v, &u, 4);
  return v;
}

// ---------------------------------------------------------------------------
// Counter PRNG: SplitMix64 output of seed + (counter+1)*gamma (nf/halfnum.py:35-45)
__device__ __forceinline__ uint64_t splitmix(uint64_t seed, uint64_t c) {
  uint64_t z = seed + (c + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// (u >> 11) * 2^-52 - 1, exact in f64 (nf/weights.py:58-62)
__device__ __forceinline__ double uniform(uint64_t seed, uint32_t stream, uint64_t i) {
  const uint64_t u = splitmix(seed, ((uint64_t)stream << 32) + i);
  return __dadd_rn(__dmul_rn((double)(u >> 11), 0x1p-52), -1.0);
}

enum SynthKind : int { K_WEIGHT = 0, K_GAIN = 1, K_LNBIAS = 2, K_BIAS = 3, K_PLAIN = 4, K_KV = 5 };

__device__ __forceinline__ double synth_value(int kind, double u, double div) {
  switch (kind) {
    case K_WEIGHT: return __ddiv_rn(u, div);                       // u / sqrt(fan_in)
    case K_GAIN: return __dadd_rn(1.0, __dmul_rn(0.1, u));         // 1 + 0.1 u
    case K_LNBIAS: return __dmul_rn(0.1, u);                       // 0.1 u
    case K_BIAS: return __dmul_rn(0.02, u);                        // 0.02 u
    case K_KV: return __dmul_rn(0.8660254037844386, u);            // var 0.25
    default: return u;
  }
}

// out[layout(i)] = fp16(synth(kind, uniform(seed, stream, i))); layout 0 row-major,
// 1 transposed, 2 8-row blocked (blk8_index)
__global__ void synth_kernel(uint64_t seed, uint32_t stream, uint64_t n, int kind, double div,
                             uint16_t* out16, float* out32, int64_t rows, int64_t cols,
                             int transpose) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint16_t hb = f64_to_f16_bits(synth_value(kind, uniform(seed, stream, i), div));
    uint64_t idx = i;
    if (transpose == 1) idx = (i % (uint64_t)cols) * (uint64_t)rows + i / (uint64_t)cols;
    else if (transpose == 2) idx = blk8_index(i / (uint64_t)cols, i % (uint64_t)cols, (size_t)cols);
    if (out16) out16[idx] = hb;
    else out32[idx] = f16_bits_to_f32(hb);
  }
}

// KV prefix [H][count][d] -> cache [H][max_seq][d]
__global__ void kv_synth_kernel(uint64_t seed, uint32_t stream, int H, int count, int d, int max_seq,
                                uint16_t* out, int head0 = 0) {
  const uint64_t n = (uint64_t)H * count * d, base = (uint64_t)head0 * count * d;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t hh = i / ((uint64_t)count * d), rem = i % ((uint64_t)count * d);
    out[hh * (uint64_t)max_seq * d + rem] =
        f64_to_f16_bits(synth_value(K_KV, uniform(seed, stream, base + i), 1.0));
  }
}

// Slice [r0, r1) x [c0, c1) of a [R][K] tensor stream (element i = r * K + c
// of the full tensor, nf/weights.py:58-62) -> fp16 / fp32, stored row-major
// or transposed within the slice (tensor-parallel shards).
__global__ void synth_slice_kernel(uint64_t seed, uint32_t stream, int64_t K, int64_t r0, int64_t r1, int64_t c0,
                                   int64_t c1, int kind, double div, uint16_t* out16, float* out32,
                                   int transpose) {
  const int64_t nr = r1 - r0, nc = c1 - c0, n = nr * nc;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = r0 + j / nc, c = c0 + j % nc;
    const uint16_t hb = f64_to_f16_bits(synth_value(kind, uniform(seed, stream, (uint64_t)(r * K + c)), div));
    const int64_t idx = transpose ? (j % nc) * nr + j / nc : j;
    if (out16) out16[idx] = hb;
    else out32[idx] = f16_bits_to_f32(hb);
  }
}

int launch_synth_slice(cudaStream_t st, uint64_t seed, uint32_t stream, int64_t K, int64_t r0, int64_t r1,
                       int64_t c0, int64_t c1, int kind, double div, uint16_t* out16, float* out32,
                       int transpose = 0) {
  synth_slice_kernel<<<148 * 16, 256, 0, st>>>(seed, stream, K, r0, r1, c0, c1, kind, div, out16, out32,
                                               transpose);
  CK(cudaGetLastError());
  return NFB_OK;
}

__global__ void set_pos_kernel(int* state, int pos) { state[0] = pos; }

__global__ void advance_state_kernel(int* state) {
  state[0] += 1;
  state[1] += 1;
}

int launch_synth(cudaStream_t st, uint64_t seed, uint32_t stream, uint64_t n, int kind, double div,
                 uint16_t* out16, float* out32, int64_t rows = 0, int64_t cols = 0, int transpose = 0) {
  const int block = 256;
  const uint64_t want = (n + block - 1) / block;
  const int grid = (int)std::min<uint64_t>(want, 148 * 32);
  synth_kernel<<<std::max(grid, 1), block, 0, st>>>(seed, stream, n, kind, div, out16, out32, rows,
                                                    cols, transpose);
  CK(cudaGetLastError());
  return NFB_OK;
}

}  // namespace

// ===========================================================================
// Context
// ===========================================================================
struct LayerBufs {
  uint16_t *wqkv = nullptr, *woT = nullptr, *wup = nullptr, *wdT = nullptr, *kc = nullptr, *vc = nullptr;
  float *bqkv = nullptr, *bo = nullptr, *bup = nullptr, *bd = nullptr;
  float *ln1g = nullptr, *ln1b = nullptr, *ln2g = nullptr, *ln2b = nullptr;
  bool weights = false;
  int kv_len = 0;
};

struct nfb_ctx {
  nfb_model_desc desc{};
  int device = 0;
  int max_seq = 0;
  int C = 2, n_clusters = 0, grid = 0, ncw = 0, block = 0, dpl = 0;  // dpl: kernel variant
  int stage_rows = 8, slot_bytes = 0, n_slots = 0, kv_pos = 0, smem = 0, sm_count = 0;
  bool coop = true;
  cudaStream_t stream = nullptr;
  std::vector<LayerBufs> layers;
  LayerW* d_layers = nullptr;
  uint16_t *embed = nullptr, *unembed = nullptr;
  float *lnfg = nullptr, *lnfb = nullptr;
  bool has_embed = false, has_unembed = false, has_lnf = false;
  float2* rope = nullptr;
  float *xs = nullptr, *rbuf = nullptr, *part = nullptr, *logits = nullptr;
  int *ctr = nullptr, *state = nullptr, *tokens = nullptr, *err = nullptr;
  int assist = 0;  // QKV assist parts per head (0: off)
  float* yg = nullptr;
  unsigned *yflag = nullptr, *epoch = nullptr;
  // tensor parallel (heads / FFN rows / vocab sharded over tp_size GPUs)
  int tp_rank = 0, tp_size = 1;
  nfb_model_desc full{};  // the unsharded model (desc holds this rank's shard)
  void* nccl = nullptr;   // ncclComm_t
  // batched decode (nfb_batch_*): B sequences at one position, tcgen05 GEMMs
  int bmax = 0, bcur = 0, bsplit = 1;
  // blocked (UMMA SW128) copies of every projection, per layer [qkv, out,
  // up, down] + the LM head (csrc/nfb_umma.cuh), rebuilt from the decode
  // kernel's copies when the weights change (wver)
  std::vector<uint16_t*> bw;  // [layer * 4 + j]
  uint16_t* blm = nullptr;
  unsigned long long wver = 1, bt_ver = 0;
  std::vector<uint16_t*> bkc, bvc;  // per layer [bmax][H][max_seq][d]
  float *bx = nullptr, *bq = nullptr, *bpart = nullptr, *blogits = nullptr;
  // blocked activation operands (hi / lo rows, n_pad of the largest batch)
  uint16_t *ba1 = nullptr, *ba2 = nullptr, *bctx = nullptr, *bg = nullptr;
  int *btok = nullptr, *bstate = nullptr;
  unsigned long long* bamax = nullptr;  // [bmax] packed argmax of the step
  int bpos = -1;
  // the MLP branch (LN2 -> up -> GELU -> down) runs on a second stream,
  // concurrently with the attention branch (the parallel residual makes them
  // independent); forked / joined with events (graph-capturable)
  cudaStream_t bstream2 = nullptr;
  cudaEvent_t bev[2] = {nullptr, nullptr};
  int bprefill_rows = 1;  // prefill attention: attn_tile_rows_kernel (NFB_PREFILL_ROWS=0: one row per block)
  int bfork = 4;  // fork point of the MLP branch (batch_token); 0 = one stream
  int bskip = 0;  // measurement only (NFB_BATCH_SKIP, results garbage): 1 MLP branch, 2 attention, 4 GEMMs
  // stream-K partials per GEMM role [qkv, out, up, down, lm] (the consumer
  // kernels sum the pieces) and the plans of the current batch
  float* uws[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  UPlan uplan[5] = {};
  int uplan_rows = 0;
  cudaGraph_t bgraph = nullptr;
  cudaGraphExec_t bgexec = nullptr;
  unsigned long long* gbar = nullptr;
  unsigned long long* amax = nullptr;
  int ctr_stride = 0;
  // pinned staging
  float *h_x = nullptr, *h_hidden = nullptr, *h_logits = nullptr;
  int* h_state = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  // serving step graphs by step parity: H2D of the input token, the decode
  // launch, D2H of the argmax slot -- one graph launch per nfb_step_token
  cudaGraphExec_t gtok[2] = {nullptr, nullptr};
  int decode_pos = -1;  // host mirror of the device position in decode mode
  int decode_step = 0;  // host mirror of the device step counter
  unsigned long long* trace = nullptr;
  int trace_stride = 0;
  int dyn_mlp = 0;
  int head_weight_pct = 130;
  int debug = 0;
  int pf_ahead = 0;  // L2 prefetcher lead (bytes); measured: no gain at C2
  int mlp_gap = 1;   // MLP pairs interleaved into the head schedule (split-phase cluster syncs)
  int fold_all = 1;  // see Params::fold_all
  int deterministic = 0;  // 1: fixed-order fold layer end (bitwise reproducible) instead of fp32 atomics
  int acc_prereduce = 1;  // atomic layer end: DSMEM cluster pre-reduce first (NFB_ACC_PREREDUCE=0: off)
  float* acc = nullptr;   // [n_layers][hidden] atomic layer-end accumulators
  int pair = 7;      // consumer stage pairing mask (1 MLP, 2 QKV, 4 W_out)
  unsigned long long* h_tok = nullptr;  // pinned [2]
  std::vector<void*> allocs;
};

namespace {

template <class T>
int dalloc(nfb_ctx* c, T** p, size_t n) {
  void* q = nullptr;
  CK(cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)));
  CK(cudaMemset(q, 0, std::max<size_t>(n, 1) * sizeof(T)));
  c->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return NFB_OK;
}

// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its predecessor runs; it griddepcontrol.wait's before
// touching the predecessor's results (csrc/nfb_batch.cu, csrc/nfb_umma.cu).
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

#define TRY(expr)              \
  do {                         \
    int r_ = (expr);           \
    if (r_ != NFB_OK) return r_; \
  } while (0)

Params base_params(nfb_ctx* c) {
  Params p{};
  const nfb_model_desc& m = c->desc;
  p.h = m.hidden;
  p.H = m.n_heads;
  p.d = m.d_head;
  p.m = m.d_mlp;
  p.rd = m.rotary_dims;
  p.V = m.vocab;
  p.max_seq = c->max_seq;
  p.eps = (float)m.ln_eps;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)m.d_head));
  p.parallel = m.parallel_residual ? 1 : 0;
  p.gelu_exact = m.gelu_exact ? 1 : 0;
  p.C = c->C;
  p.n_clusters = c->n_clusters;
  p.ncw = c->ncw;
  p.rows_qkv = 3 * m.d_head / (c->C + c->assist);
  p.rows_o = m.d_head / c->C;  // (average; rank r applies rows [r d / C, (r + 1) d / C))
  p.stage_rows = c->stage_rows;
  p.n_slots = c->n_slots;
  p.slot_bytes = c->slot_bytes;
  p.kv_pos = c->kv_pos;
  p.layers = c->d_layers;
  p.head.embed = reinterpret_cast<const __half*>(c->embed);
  p.head.lnfg = c->lnfg;
  p.head.lnfb = c->lnfb;
  p.head.unembed = reinterpret_cast<const __half*>(c->unembed);
  p.rope = c->rope;
  p.xs = c->xs;
  p.rbuf = c->rbuf;
  p.part = c->part;
  p.ctr = c->ctr;
  p.ctr_stride = c->ctr_stride;
  p.gbar = c->gbar;
  p.state = c->state;
  p.amax = c->amax;
  p.tokens = c->tokens;
  p.logits = c->logits;
  p.err = c->err;
  p.assist = c->assist;
  p.yg = c->yg;
  p.yflag = c->yflag;
  p.epoch = c->epoch;
  p.trace = c->trace;
  p.trace_stride = c->trace_stride;
  p.dyn_mlp = c->dyn_mlp;
  p.head_weight_pct = c->head_weight_pct;
  p.pf_ahead = c->pf_ahead;
  p.mlp_gap = c->mlp_gap;
  p.pair = (c->dpl & 1) ? (c->pair & 1) : c->pair;  // two-chunk variant: MLP pairs only (compiled out)
  p.fold_all = c->fold_all;
  p.acc = c->acc;
  p.acc_mode = (m.parallel_residual && c->tp_size == 1 && !c->deterministic) ? 1 : 0;
  p.acc_prereduce = c->acc_prereduce;
  p.tp_root = c->tp_rank == 0 ? 1 : 0;
  p.state_update = 1;
  p.vocab_offset = c->tp_rank * c->desc.vocab;
  p.vocab_full = c->full.vocab;
  p.debug = c->debug;
  return p;
}

// The lean production kernel variant has only the default path; tracing,
// debug modes and the experimental options run on the full variant.
bool needs_full_variant(const nfb_ctx* c);
// Production variants compiled for the headline shapes (row strides, warp
// counts and head size as immediates): 4 = hidden 2560 / d_head 80 (Pythia-2.8B),
// 5 = hidden 4096 / d_head 128 (Pythia-6.9B); else the runtime-shape variant.
int kernel_variant(const nfb_ctx* c) {
  if (needs_full_variant(c)) return c->dpl + 2;
  const int h = c->desc.hidden, d = c->desc.d_head;
  if (c->dpl == 0 && h == 2560 && d == 80 && c->ncw == 10) return 4;
  if (c->dpl == 1 && h == 4096 && d == 128 && c->ncw == 8) return 5;
  return c->dpl;
}

bool needs_full_variant(const nfb_ctx* c) {
  // the lean variant: parallel residual with the atomic layer end only
  const bool acc_mode = c->desc.parallel_residual && c->tp_size == 1 && !c->deterministic;
  return c->trace || c->debug || c->assist || c->pf_ahead > 0 || c->dyn_mlp || !c->fold_all || !acc_mode ||
         !c->acc_prereduce;
}

int launch(nfb_ctx* c, const Params& p, cudaStream_t st) {
  const int variant = kernel_variant(c);
  cudaError_t e = launch_decode(p, variant, c->grid, c->block, c->smem, st, c->coop);
  if (e != cudaSuccess && c->coop) {
    // Cooperative + cluster launch refused: fall back to the occupancy-checked
    // plain cluster launch (grid <= max active clusters, one CTA per SM).
    cudaGetLastError();
    c->coop = false;
    e = launch_decode(p, variant, c->grid, c->block, c->smem, st, false);
  }
  if (e != cudaSuccess) return fail(NFB_ECUDA, std::string("decode launch: ") + cudaGetErrorString(e));
  return NFB_OK;
}

}  // namespace

// One decode token under tensor parallelism: per layer a launch that leaves
// this rank's split-K partial (rank 0: + residual + biases) in xs[l+1], then
// an NCCL sum all-reduce of that [h] vector; the vocab-sharded LM head; a max
// all-reduce of the packed (logit, ~index) argmax slots; the (pos, step)
// advance.  Graph-capturable (NCCL supports stream capture).
static int tp_token(nfb_ctx* c, cudaStream_t st) {
  if (!c->nccl) return fail(NFB_ESTATE, "tensor-parallel context: call nfb_tp_init first");
  if (c->trace || c->debug) return fail(NFB_EUNSUPPORTED, "tracing is single-launch only");
  NcclApi& n = nccl_api();
  const int L = c->desc.n_layers, h = c->desc.hidden;
  for (int l = 0; l < L; ++l) {
    Params p = base_params(c);
    p.l0 = l;
    p.l1 = l + 1;
    p.xs = c->xs + (size_t)l * h;
    p.in_mode = l == 0 ? IN_TOKEN : IN_X;
    p.head_mode = HEAD_NONE;
    p.advance_pos = 0;
    p.state_update = 0;
    TRY(launch(c, p, st));
    NCK(n.allReduce(c->xs + (size_t)(l + 1) * h, c->xs + (size_t)(l + 1) * h, (size_t)h, ncclFloat32, ncclSum,
                    (ncclComm_t)c->nccl, st));
  }
  Params p = base_params(c);
  p.l0 = p.l1 = L;
  p.xs = c->xs + (size_t)L * h;
  p.in_mode = IN_X;
  p.head_mode = HEAD_LM;
  p.advance_pos = 0;
  p.state_update = 0;
  TRY(launch(c, p, st));
  // both parity slots: the other one already holds identical values on every rank
  NCK(n.allReduce(c->amax, c->amax, 2, ncclUint64, ncclMax, (ncclComm_t)c->nccl, st));
  advance_state_kernel<<<1, 1, 0, st>>>(c->state);
  CK(cudaGetLastError());
  return NFB_OK;
}

namespace {

// Zero both parities of the dynamic row counters (LM-head rows, dynamic MLP
// chunks).  In graph / decode mode the kernel keeps them consistent by step
// parity; every launch that does not advance the step (block step, forward,
// head logits) or that rewinds it (begin_decode) must start from zero, or a
// parity slot exhausted by an earlier launch hands out no rows.
int reset_counters(nfb_ctx* c, cudaStream_t st) {
  CK(cudaMemsetAsync(c->ctr, 0, sizeof(int) * 2 * (size_t)c->ctr_stride, st));
  // the atomic layer-end accumulators are all zero between launches (the
  // kernel re-zeroes them); re-establish that after a rewind or a fault
  CK(cudaMemsetAsync(c->acc, 0, sizeof(float) * (size_t)c->desc.n_layers * c->desc.hidden, st));
  return NFB_OK;
}

int check_device_error(nfb_ctx* c) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    int code = 0;
    cudaMemcpy(&code, c->err, sizeof(int), cudaMemcpyDeviceToHost);
    return fail(NFB_EDEVICE, std::string("device failure (watchdog code ") + std::to_string(code) +
                                 "): " + cudaGetErrorString(e));
  }
  return NFB_OK;
}

int to_f16_host(const void* src, int dtype, size_t n, std::vector<uint16_t>& out) {
  out.resize(n);
  if (dtype == NFB_F64) {
    const double* s = static_cast<const double*>(src);
    for (size_t i = 0; i < n; ++i) out[i] = f64_to_f16_bits(s[i]);
  } else if (dtype == NFB_F32) {
    const float* s = static_cast<const float*>(src);
    for (size_t i = 0; i < n; ++i) out[i] = f64_to_f16_bits((double)s[i]);
  } else if (dtype == NFB_F16) {
    memcpy(out.data(), src, n * 2);
  } else {
    return fail(NFB_EINVAL, "dtype must be NFB_F64, NFB_F32 or NFB_F16");
  }
  return NFB_OK;
}

enum Layout2D : int { L_ROW = 0, L_TRANSPOSED = 1, L_BLK8 = 2 };

size_t layout_index(int layout, size_t r, size_t k, size_t rows, size_t cols) {
  if (layout == L_TRANSPOSED) return k * rows + r;
  if (layout == L_BLK8) return blk8_index(r, k, cols);
  return r * cols + k;
}

int upload_f16(const void* src, int dtype, size_t rows, size_t cols, int layout, uint16_t* dst) {
  std::vector<uint16_t> h;
  TRY(to_f16_host(src, dtype, rows * cols, h));
  if (layout != L_ROW) {
    std::vector<uint16_t> t(rows * cols);
    for (size_t r = 0; r < rows; ++r)
      for (size_t k = 0; k < cols; ++k) t[layout_index(layout, r, k, rows, cols)] = h[r * cols + k];
    h.swap(t);
  }
  CK(cudaMemcpy(dst, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  return NFB_OK;
}

int upload_f32_of_f16(const void* src, int dtype, size_t n, float* dst) {
  std::vector<uint16_t> h;
  TRY(to_f16_host(src, dtype, n, h));
  std::vector<float> f(n);
  for (size_t i = 0; i < n; ++i) f[i] = f16_bits_to_f32(h[i]);
  CK(cudaMemcpy(dst, f.data(), n * 4, cudaMemcpyHostToDevice));
  return NFB_OK;
}

int check_layer(nfb_ctx* c, int layer) {
  if (!c) return fail(NFB_EINVAL, "null context");
  if (layer < 0 || layer >= c->desc.n_layers)
    return fail(NFB_EINVAL, "layer " + std::to_string(layer) + " out of range");
  return NFB_OK;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
// nfb_create / nfb_create_tp: `full` is the unsharded model (== desc unless
// tensor parallel, where desc holds this rank's heads / FFN rows / vocab).
static int create_ctx(const nfb_model_desc* desc, const nfb_model_desc* full, int device, int max_seq,
                      int cluster_size, int max_clusters, nfb_ctx** out);

extern "C" {

int nfb_version(void) { return 100; }

const char* nfb_last_error(void) { return g_err.c_str(); }

int nfb_create(const nfb_model_desc* desc, int device, int max_seq, int cluster_size,
               int max_clusters, nfb_ctx** out) {
  return create_ctx(desc, desc, device, max_seq, cluster_size, max_clusters, out);
}
}  // extern "C"

static int create_ctx(const nfb_model_desc* desc, const nfb_model_desc* full, int device, int max_seq,
                      int cluster_size, int max_clusters, nfb_ctx** out) {
  if (!desc || !out) return fail(NFB_EINVAL, "null argument");
  *out = nullptr;
  const nfb_model_desc& m = *desc;
  if (m.hidden < 1 || m.n_heads < 1 || m.d_head < 1 || m.n_layers < 1 || m.d_mlp < 1 || m.vocab < 1)
    return fail(NFB_EINVAL, "model dimensions must be >= 1");
  if (m.hidden != m.n_heads * m.d_head && desc == full)
    return fail(NFB_EINVAL, "hidden (" + std::to_string(m.hidden) + ") must equal n_heads * d_head (" +
                                std::to_string(m.n_heads) + " * " + std::to_string(m.d_head) + ")");
  if (m.rotary_dims < 2 || m.rotary_dims % 2 || m.rotary_dims > m.d_head)
    return fail(NFB_EINVAL, "rotary_dims must be an even number >= 2 and <= d_head");
  if (!(m.ln_eps > 0.0)) return fail(NFB_EINVAL, "ln_eps must be positive");
  if (m.hidden % 8 || m.hidden > 32 * 8 * kMaxConsumerWarps)
    return fail(NFB_EUNSUPPORTED, "hidden must be a multiple of 8 and <= 4096");
  if (m.d_head % 8) return fail(NFB_EUNSUPPORTED, "d_head must be a multiple of 8");
  if (max_seq < 1) return fail(NFB_EINVAL, "max_seq must be >= 1");
  // Default cluster size: 2 CTAs per head; 3 once a head's KV history
  // (4 d bytes per position) outweighs ~40 % of its serial chain (QKV +
  // W_out rows, 8 d h bytes): max_seq > 4 h / 3.  Measured, C = 2 vs 3:
  // Pythia-2.8B ctx 1024 952 vs 884, 3072 799 vs 804, 4096 709 vs 782, 8192
  // 535 vs 653 tok/s; Pythia-6.9B ctx 4096 345 vs 325 (threshold 5461).
  int C = cluster_size > 0 ? cluster_size : 2;
  if (cluster_size <= 0 && 3LL * max_seq > 4LL * m.hidden && (m.d_head % 4) == 0) C = 3;
  if (cluster_size <= 0 && getenv("NFB_CLUSTER")) C = atoi(getenv("NFB_CLUSTER"));
  if (C > 8 || (3 * m.d_head) % C || ((3 * m.d_head) / C) % 4)
    return fail(NFB_EUNSUPPORTED, "cluster_size must be <= 8 and leave an equal multiple of 4 QKV rows per rank");

  nfb_ctx* c = new nfb_ctx();
  c->desc = m;
  c->full = *full;
  c->device = device;
  c->max_seq = max_seq;
  c->C = C;
  auto bail = [&](int code) {
    nfb_destroy(c);
    return code;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return bail(fail(NFB_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)));
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return bail(fail(NFB_ECUDA, cudaGetErrorString(e)));

  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  c->sm_count = prop.multiProcessorCount;
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);

  // consumer thread t owns 16-byte hidden chunks t (+ nct for 2 chunks/thread)
  const int nch = m.hidden / 8 > 320 ? 2 : 1;
  c->ncw = (m.hidden / 8 / nch + 31) / 32;
  c->block = (c->ncw + 2) * 32;  // consumers + ring producer warp + L2 prefetcher warp
  c->dpl = nch - 1;              // kernel variant (chunks per consumer thread)
  c->stage_rows = kRows;  // 8-row stages (64 KB at hidden 4096: 3 ring slots)
  if (getenv("NFB_STAGE_ROWS")) c->stage_rows = std::max(1, std::min(kRows, atoi(getenv("NFB_STAGE_ROWS"))));
  c->slot_bytes = std::max(c->stage_rows * m.hidden * 2, 4 * m.d_head * 2 * 2);
  c->kv_pos = c->slot_bytes / (4 * m.d_head);
  Params probe = base_params(c);
  probe.n_slots = 0;
  const int fixed = make_layout(probe).total;
  const int per_slot = c->slot_bytes + 32;
  c->n_slots = std::min(12, (smem_optin - fixed - 128) / per_slot);
  if (c->n_slots < 2) return bail(fail(NFB_EUNSUPPORTED, "shared memory too small for the stage ring"));
  probe.n_slots = c->n_slots;
  c->smem = make_layout(probe).total;

  e = cudaSuccess;
  for (int v : {c->dpl, c->dpl + 2, 4 + c->dpl})  // runtime-shape, full, and headline-shape variants
    if (e == cudaSuccess) e = cudaFuncSetAttribute(decode_kernel_ptr(v), cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem);
  if (e != cudaSuccess) return bail(fail(NFB_ECUDA, std::string("smem attribute: ") + cudaGetErrorString(e)));
  int nc = 0;
  e = max_active_clusters(c->dpl, C, c->block, c->smem, &nc);
  if (e != cudaSuccess || nc < 1)
    return bail(fail(NFB_ECUDA, std::string("no co-resident cluster fits: ") + cudaGetErrorString(e)));
  if (max_clusters <= 0 && getenv("NFB_MAX_CLUSTERS")) max_clusters = atoi(getenv("NFB_MAX_CLUSTERS"));
  if (max_clusters > 0) nc = std::min(nc, max_clusters);
  // Plain cluster launch (grid <= max co-resident clusters, one CTA per SM:
  // still co-resident) on request or under Nsight Compute, whose kernel
  // replay does not support cooperative launches (the driver's ncu pass
  // reported rc 9 / no time for the cooperative launch).
  if (getenv("NFB_NO_COOP") || getenv("CUDA_INJECTION64_PATH") || getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE"))
    c->coop = false;
  if (getenv("NFB_HEAD_WEIGHT")) c->head_weight_pct = atoi(getenv("NFB_HEAD_WEIGHT"));
  if (getenv("NFB_DEBUG")) c->debug = atoi(getenv("NFB_DEBUG"));
  if (getenv("NFB_PREFETCH_KB")) c->pf_ahead = atoi(getenv("NFB_PREFETCH_KB")) * 1024;
  if (getenv("NFB_MLP_GAP")) c->mlp_gap = atoi(getenv("NFB_MLP_GAP"));
  // QKV / W_out pairs pay at one chunk per thread (C2: +1.9 %) but cost the
  // two-chunk variant registers (C3 at weight 80: 294 vs 335 tok/s)
  if (c->dpl & 1) c->pair = 1;
  if (getenv("NFB_PAIR")) c->pair = atoi(getenv("NFB_PAIR"));
  if (getenv("NFB_FOLD_ALL")) c->fold_all = atoi(getenv("NFB_FOLD_ALL")) ? 1 : 0;
  if (getenv("NFB_DETERMINISTIC")) c->deterministic = atoi(getenv("NFB_DETERMINISTIC")) ? 1 : 0;
  if (getenv("NFB_ACC_PREREDUCE")) c->acc_prereduce = atoi(getenv("NFB_ACC_PREREDUCE")) ? 1 : 0;
  if (getenv("NFB_ASSIST")) c->assist = atoi(getenv("NFB_ASSIST"));
  if (getenv("NFB_DYN_MLP")) c->dyn_mlp = atoi(getenv("NFB_DYN_MLP")) ? 1 : 0;
  // assist needs CTAs without heads, parts of a multiple of 4 rows, <= 8 parts
  if (c->assist < 0 || c->assist > 6 || (3 * m.d_head) % (C + c->assist) || ((3 * m.d_head) / (C + c->assist)) % 4 ||
      nc * C <= C * std::min(m.n_heads, nc))
    c->assist = 0;
  c->n_clusters = nc;
  c->grid = nc * C;

  const int L = m.n_layers, h = m.hidden, H = m.n_heads, d = m.d_head, mm = m.d_mlp, V = m.vocab;
  c->layers.resize(L);
  std::vector<LayerW> table(L);
  for (int l = 0; l < L; ++l) {
    LayerBufs& b = c->layers[l];
    int r = NFB_OK;
    if ((r = dalloc(c, &b.wqkv, (size_t)3 * h * h)) || (r = dalloc(c, &b.woT, (size_t)h * h)) ||
        (r = dalloc(c, &b.wup, (size_t)mm * h)) || (r = dalloc(c, &b.wdT, (size_t)mm * h)) ||
        (r = dalloc(c, &b.bqkv, (size_t)3 * h)) || (r = dalloc(c, &b.bo, h)) ||
        (r = dalloc(c, &b.bup, mm)) || (r = dalloc(c, &b.bd, h)) || (r = dalloc(c, &b.ln1g, h)) ||
        (r = dalloc(c, &b.ln1b, h)) || (r = dalloc(c, &b.ln2g, h)) || (r = dalloc(c, &b.ln2b, h)) ||
        (r = dalloc(c, &b.kc, (size_t)H * max_seq * d)) || (r = dalloc(c, &b.vc, (size_t)H * max_seq * d)))
      return bail(r);
    LayerW& w = table[l];
    w.wqkv = reinterpret_cast<const __half*>(b.wqkv);
    w.woT = reinterpret_cast<const __half*>(b.woT);
    w.wup = reinterpret_cast<const __half*>(b.wup);
    w.wdT = reinterpret_cast<const __half*>(b.wdT);
    w.bqkv = b.bqkv;
    w.bo = b.bo;
    w.bup = b.bup;
    w.bd = b.bd;
    w.ln1g = b.ln1g;
    w.ln1b = b.ln1b;
    w.ln2g = b.ln2g;
    w.ln2b = b.ln2b;
    w.kc = reinterpret_cast<__half*>(b.kc);
    w.vc = reinterpret_cast<__half*>(b.vc);
  }
  int r = NFB_OK;
  c->ctr_stride = L + 2;
  if ((r = dalloc(c, &c->d_layers, L)) || (r = dalloc(c, &c->embed, (size_t)c->full.vocab * h)) ||
      (r = dalloc(c, &c->unembed, (size_t)V * h)) || (r = dalloc(c, &c->lnfg, h)) ||
      (r = dalloc(c, &c->lnfb, h)) || (r = dalloc(c, &c->rope, (size_t)max_seq * (m.rotary_dims / 2))) ||
      (r = dalloc(c, &c->xs, (size_t)(L + 1) * h)) || (r = dalloc(c, &c->rbuf, h)) ||
      (r = dalloc(c, &c->part, (size_t)nc * C * h)) || (r = dalloc(c, &c->acc, (size_t)L * h)) ||
      (r = dalloc(c, &c->logits, V)) ||
      (r = dalloc(c, &c->ctr, 2 * c->ctr_stride)) || (r = dalloc(c, &c->gbar, 2)) ||
      (r = dalloc(c, &c->state, 2)) || (r = dalloc(c, &c->amax, 2)) ||
      (r = dalloc(c, &c->tokens, max_seq)) || (r = dalloc(c, &c->err, 1)) ||
      (r = dalloc(c, &c->yg, (size_t)H * 3 * d)) || (r = dalloc(c, &c->yflag, (size_t)H * 8)) ||
      (r = dalloc(c, &c->epoch, 1)))
    return bail(r);
  e = cudaMemcpy(c->d_layers, table.data(), sizeof(LayerW) * L, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return bail(fail(NFB_ECUDA, cudaGetErrorString(e)));

  // RoPE table: angle = pos * base^(-2i/rd) in f64 (nf/golden.py:68-71), cos/sin -> fp32
  const int half = m.rotary_dims / 2;
  std::vector<float2> rope((size_t)max_seq * half);
  for (int pos = 0; pos < max_seq; ++pos)
    for (int i = 0; i < half; ++i) {
      const double th = pos * std::pow(m.theta_base, -2.0 * i / m.rotary_dims);
      rope[(size_t)pos * half + i] = make_float2((float)std::cos(th), (float)std::sin(th));
    }
  e = cudaMemcpy(c->rope, rope.data(), rope.size() * sizeof(float2), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return bail(fail(NFB_ECUDA, cudaGetErrorString(e)));

  if (cudaMallocHost(&c->h_x, (size_t)h * 4) != cudaSuccess ||
      cudaMallocHost(&c->h_hidden, (size_t)(L + 1) * h * 4) != cudaSuccess ||
      cudaMallocHost(&c->h_logits, (size_t)V * 4) != cudaSuccess ||
      cudaMallocHost(&c->h_state, 4 * sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&c->h_tok, 2 * sizeof(unsigned long long)) != cudaSuccess)
    return bail(fail(NFB_ECUDA, "pinned host staging allocation failed"));
  *out = c;
  return NFB_OK;
}

extern "C" {

int nfb_destroy(nfb_ctx* c) {
  if (!c) return NFB_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->nccl && nccl_api().ok) nccl_api().commDestroy((ncclComm_t)c->nccl);
  if (c->bgexec) cudaGraphExecDestroy(c->bgexec);
  if (c->bgraph) cudaGraphDestroy(c->bgraph);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  for (auto& g : c->gtok)
    if (g) cudaGraphExecDestroy(g);
  if (c->graph) cudaGraphDestroy(c->graph);
  for (void* p : c->allocs) cudaFree(p);
  if (c->h_x) cudaFreeHost(c->h_x);
  if (c->h_hidden) cudaFreeHost(c->h_hidden);
  if (c->h_logits) cudaFreeHost(c->h_logits);
  if (c->h_state) cudaFreeHost(c->h_state);
  if (c->h_tok) cudaFreeHost(c->h_tok);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->bstream2) cudaStreamDestroy(c->bstream2);
  for (auto& e : c->bev)
    if (e) cudaEventDestroy(e);
  delete c;
  return NFB_OK;
}

int nfb_get_info(nfb_ctx* c, nfb_info* info) {
  if (!c || !info) return fail(NFB_EINVAL, "null argument");
  info->grid = c->grid;
  info->cluster_size = c->C;
  info->n_clusters = c->n_clusters;
  info->consumer_warps = c->ncw;
  info->stage_rows = c->stage_rows;
  info->n_slots = c->n_slots;
  info->slot_bytes = c->slot_bytes;
  info->kv_stage_pos = c->kv_pos;
  info->smem_bytes = c->smem;
  info->max_seq = c->max_seq;
  info->sm_count = c->sm_count;
  return NFB_OK;
}

void* nfb_stream(nfb_ctx* c) { return c ? (void*)c->stream : nullptr; }

int nfb_set_block_weights(nfb_ctx* c, int layer, const nfb_block_weights* w, int dtype) {
  TRY(check_layer(c, layer));
  ++c->wver;
  if (c->tp_size > 1) return fail(NFB_EUNSUPPORTED, "tensor-parallel contexts take synthesized weights");
  if (!w) return fail(NFB_EINVAL, "null weights");
  const void* ptrs[12] = {w->ln1_gain, w->ln1_bias, w->qkv_weight, w->qkv_bias, w->out_weight, w->out_bias,
                          w->ln2_gain, w->ln2_bias, w->up_weight, w->up_bias, w->down_weight, w->down_bias};
  for (const void* p : ptrs)
    if (!p) return fail(NFB_EINVAL, "every BlockWeights tensor is required");
  cudaSetDevice(c->device);
  CK(cudaStreamSynchronize(c->stream));  // legacy-stream copies below: order after queued launches
  const int h = c->desc.hidden, m = c->desc.d_mlp;
  LayerBufs& b = c->layers[layer];
  TRY(upload_f32_of_f16(w->ln1_gain, dtype, h, b.ln1g));
  TRY(upload_f32_of_f16(w->ln1_bias, dtype, h, b.ln1b));
  TRY(upload_f16(w->qkv_weight, dtype, (size_t)3 * h, h, L_ROW, b.wqkv));
  TRY(upload_f32_of_f16(w->qkv_bias, dtype, (size_t)3 * h, b.bqkv));
  TRY(upload_f16(w->out_weight, dtype, h, h, L_TRANSPOSED, b.woT));
  TRY(upload_f32_of_f16(w->out_bias, dtype, h, b.bo));
  TRY(upload_f32_of_f16(w->ln2_gain, dtype, h, b.ln2g));
  TRY(upload_f32_of_f16(w->ln2_bias, dtype, h, b.ln2b));
  TRY(upload_f16(w->up_weight, dtype, m, h, L_ROW, b.wup));
  TRY(upload_f32_of_f16(w->up_bias, dtype, m, b.bup));
  TRY(upload_f16(w->down_weight, dtype, h, m, L_TRANSPOSED, b.wdT));
  TRY(upload_f32_of_f16(w->down_bias, dtype, h, b.bd));
  b.weights = true;
  return NFB_OK;
}

int nfb_synth_block_weights(nfb_ctx* c, int layer, uint64_t seed) {
  TRY(check_layer(c, layer));
  ++c->wver;
  cudaSetDevice(c->device);
  const int64_t h = c->desc.hidden, m = c->desc.d_mlp;
  LayerBufs& b = c->layers[layer];
  cudaStream_t st = c->stream;
  if (c->tp_size > 1) {
    // this rank's shard of the full layer's streams: heads [hs, he), MLP rows [ms, me)
    const int64_t d = c->desc.d_head, H = c->desc.n_heads, M = c->full.d_mlp;
    const int64_t hs = c->tp_rank * H, he = hs + H, ms = c->tp_rank * m, me = ms + m;
    const double sh = std::sqrt((double)h), sm = std::sqrt((double)M);
    TRY(launch_synth(st, seed, 0, h, K_GAIN, 1.0, nullptr, b.ln1g));
    TRY(launch_synth(st, seed, 1, h, K_LNBIAS, 1.0, nullptr, b.ln1b));
    TRY(launch_synth_slice(st, seed, 2, h, hs * 3 * d, he * 3 * d, 0, h, K_WEIGHT, sh, b.wqkv, nullptr));
    TRY(launch_synth_slice(st, seed, 3, 3 * h, 0, 1, hs * 3 * d, he * 3 * d, K_BIAS, 1.0, nullptr, b.bqkv));
    TRY(launch_synth_slice(st, seed, 4, h, 0, h, hs * d, he * d, K_WEIGHT, sh, b.woT, nullptr, 1));
    TRY(launch_synth(st, seed, 5, h, K_BIAS, 1.0, nullptr, b.bo));
    TRY(launch_synth(st, seed, 6, h, K_GAIN, 1.0, nullptr, b.ln2g));
    TRY(launch_synth(st, seed, 7, h, K_LNBIAS, 1.0, nullptr, b.ln2b));
    TRY(launch_synth_slice(st, seed, 8, h, ms, me, 0, h, K_WEIGHT, sh, b.wup, nullptr));
    TRY(launch_synth_slice(st, seed, 9, M, 0, 1, ms, me, K_BIAS, 1.0, nullptr, b.bup));
    TRY(launch_synth_slice(st, seed, 10, M, 0, h, ms, me, K_WEIGHT, sm, b.wdT, nullptr, 1));
    TRY(launch_synth(st, seed, 11, h, K_BIAS, 1.0, nullptr, b.bd));
    CK(cudaStreamSynchronize(st));
    b.weights = true;
    return NFB_OK;
  }
  // stream index = position in BlockWeights field order (nf/weights.py:55, 80-82)
  TRY(launch_synth(st, seed, 0, h, K_GAIN, 1.0, nullptr, b.ln1g));
  TRY(launch_synth(st, seed, 1, h, K_LNBIAS, 1.0, nullptr, b.ln1b));
  TRY(launch_synth(st, seed, 2, 3 * h * h, K_WEIGHT, std::sqrt((double)h), b.wqkv, nullptr));
  TRY(launch_synth(st, seed, 3, 3 * h, K_BIAS, 1.0, nullptr, b.bqkv));
  TRY(launch_synth(st, seed, 4, h * h, K_WEIGHT, std::sqrt((double)h), b.woT, nullptr, h, h, L_TRANSPOSED));
  TRY(launch_synth(st, seed, 5, h, K_BIAS, 1.0, nullptr, b.bo));
  TRY(launch_synth(st, seed, 6, h, K_GAIN, 1.0, nullptr, b.ln2g));
  TRY(launch_synth(st, seed, 7, h, K_LNBIAS, 1.0, nullptr, b.ln2b));
  TRY(launch_synth(st, seed, 8, m * h, K_WEIGHT, std::sqrt((double)h), b.wup, nullptr));
  TRY(launch_synth(st, seed, 9, m, K_BIAS, 1.0, nullptr, b.bup));
  TRY(launch_synth(st, seed, 10, h * m, K_WEIGHT, std::sqrt((double)m), b.wdT, nullptr, h, m, L_TRANSPOSED));
  TRY(launch_synth(st, seed, 11, h, K_BIAS, 1.0, nullptr, b.bd));
  CK(cudaStreamSynchronize(st));
  b.weights = true;
  return NFB_OK;
}

static int read_f16(const uint16_t* src, size_t rows, size_t cols, int layout, void* dst) {
  std::vector<uint16_t> h(rows * cols);
  CK(cudaMemcpy(h.data(), src, h.size() * 2, cudaMemcpyDeviceToHost));
  float* o = static_cast<float*>(dst);
  for (size_t r = 0; r < rows; ++r)
    for (size_t k = 0; k < cols; ++k) o[r * cols + k] = f16_bits_to_f32(h[layout_index(layout, r, k, rows, cols)]);
  return NFB_OK;
}

static int read_f32(const float* src, size_t n, void* dst) {
  CK(cudaMemcpy(dst, src, n * 4, cudaMemcpyDeviceToHost));
  return NFB_OK;
}

int nfb_read_block_weights(nfb_ctx* c, int layer, const nfb_block_weights* w) {
  TRY(check_layer(c, layer));
  if (!w) return fail(NFB_EINVAL, "null weights");
  cudaSetDevice(c->device);
  CK(cudaStreamSynchronize(c->stream));
  const size_t h = c->desc.hidden, m = c->desc.d_mlp;
  LayerBufs& b = c->layers[layer];
  void* o[12] = {(void*)w->ln1_gain, (void*)w->ln1_bias, (void*)w->qkv_weight, (void*)w->qkv_bias,
                 (void*)w->out_weight, (void*)w->out_bias, (void*)w->ln2_gain, (void*)w->ln2_bias,
                 (void*)w->up_weight, (void*)w->up_bias, (void*)w->down_weight, (void*)w->down_bias};
  for (void* p : o)
    if (!p) return fail(NFB_EINVAL, "every output tensor is required");
  TRY(read_f32(b.ln1g, h, o[0]));
  TRY(read_f32(b.ln1b, h, o[1]));
  TRY(read_f16(b.wqkv, 3 * h, h, L_ROW, o[2]));
  TRY(read_f32(b.bqkv, 3 * h, o[3]));
  TRY(read_f16(b.woT, h, h, L_TRANSPOSED, o[4]));
  TRY(read_f32(b.bo, h, o[5]));
  TRY(read_f32(b.ln2g, h, o[6]));
  TRY(read_f32(b.ln2b, h, o[7]));
  TRY(read_f16(b.wup, m, h, L_ROW, o[8]));
  TRY(read_f32(b.bup, m, o[9]));
  TRY(read_f16(b.wdT, h, m, L_TRANSPOSED, o[10]));
  TRY(read_f32(b.bd, h, o[11]));
  return NFB_OK;
}

int nfb_set_head(nfb_ctx* c, const void* embed, const void* lnf_gain, const void* lnf_bias,
                 const void* unembed, int dtype) {
  if (!c) return fail(NFB_EINVAL, "null context");
  if (c->tp_size > 1) return fail(NFB_EUNSUPPORTED, "tensor-parallel contexts take synthesized weights");
  cudaSetDevice(c->device);
  CK(cudaStreamSynchronize(c->stream));
  const size_t h = c->desc.hidden, V = c->desc.vocab;
  if (embed) {
    TRY(upload_f16(embed, dtype, V, h, L_ROW, c->embed));
    c->has_embed = true;
  }
  if (lnf_gain || lnf_bias) {
    if (!lnf_gain || !lnf_bias) return fail(NFB_EINVAL, "final LN needs gain and bias");
    TRY(upload_f32_of_f16(lnf_gain, dtype, h, c->lnfg));
    TRY(upload_f32_of_f16(lnf_bias, dtype, h, c->lnfb));
    c->has_lnf = true;
  }
  if (unembed) {
    TRY(upload_f16(unembed, dtype, V, h, L_ROW, c->unembed));
    c->has_unembed = true;
    ++c->wver;  // the batched path's blocked LM-head copy
  }
  return NFB_OK;
}

int nfb_synth_head(nfb_ctx* c, uint64_t seed) {
  if (!c) return fail(NFB_EINVAL, "null context");
  cudaSetDevice(c->device);
  const int64_t h = c->desc.hidden, V = c->desc.vocab;
  cudaStream_t st = c->stream;
  // the embedding table is replicated (full vocab); the unembedding is this
  // rank's vocab shard under tensor parallelism
  TRY(launch_synth(st, seed, 0, (int64_t)c->full.vocab * h, K_PLAIN, 1.0, c->embed, nullptr));
  TRY(launch_synth(st, seed, 1, h, K_GAIN, 1.0, nullptr, c->lnfg));
  TRY(launch_synth(st, seed, 2, h, K_LNBIAS, 1.0, nullptr, c->lnfb));
  TRY(launch_synth_slice(st, seed, 3, h, (int64_t)c->tp_rank * V, (int64_t)(c->tp_rank + 1) * V, 0, h, K_WEIGHT,
                         std::sqrt((double)h), c->unembed, nullptr));
  CK(cudaStreamSynchronize(st));
  c->has_embed = c->has_lnf = c->has_unembed = true;
  ++c->wver;
  return NFB_OK;
}

int nfb_kv_write(nfb_ctx* c, int layer, int start, int count, const void* keys, const void* values,
                 int dtype) {
  TRY(check_layer(c, layer));
  LayerBufs& b = c->layers[layer];
  if (start < 0 || count < 0 || start > b.kv_len || start + count > c->max_seq)
    return fail(NFB_EINVAL, "KV write range [" + std::to_string(start) + ", " + std::to_string(start + count) +
                                ") invalid for a cache holding " + std::to_string(b.kv_len) +
                                " positions (capacity " + std::to_string(c->max_seq) + ")");
  if (count && (!keys || !values)) return fail(NFB_EINVAL, "null keys/values");
  cudaSetDevice(c->device);
  CK(cudaStreamSynchronize(c->stream));
  const size_t H = c->desc.n_heads, d = c->desc.d_head;
  if (count) {
    std::vector<uint16_t> hk, hv;
    TRY(to_f16_host(keys, dtype, H * count * d, hk));
    TRY(to_f16_host(values, dtype, H * count * d, hv));
    CK(cudaMemcpy2D(b.kc + (size_t)start * d, c->max_seq * d * 2, hk.data(), (size_t)count * d * 2,
                    (size_t)count * d * 2, H, cudaMemcpyHostToDevice));
    CK(cudaMemcpy2D(b.vc + (size_t)start * d, c->max_seq * d * 2, hv.data(), (size_t)count * d * 2,
                    (size_t)count * d * 2, H, cudaMemcpyHostToDevice));
  }
  b.kv_len = start + count;
  return NFB_OK;
}

int nfb_kv_read(nfb_ctx* c, int layer, int start, int count, float* keys, float* values) {
  TRY(check_layer(c, layer));
  LayerBufs& b = c->layers[layer];
  if (start < 0 || count < 0 || start + count > c->max_seq) return fail(NFB_EINVAL, "KV read range invalid");
  cudaSetDevice(c->device);
  CK(cudaStreamSynchronize(c->stream));
  const size_t H = c->desc.n_heads, d = c->desc.d_head;
  std::vector<uint16_t> hk(H * count * d), hv(H * count * d);
  if (count) {
    CK(cudaMemcpy2D(hk.data(), (size_t)count * d * 2, b.kc + (size_t)start * d, c->max_seq * d * 2,
                    (size_t)count * d * 2, H, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy2D(hv.data(), (size_t)count * d * 2, b.vc + (size_t)start * d, c->max_seq * d * 2,
                    (size_t)count * d * 2, H, cudaMemcpyDeviceToHost));
  }
  for (size_t i = 0; i < hk.size(); ++i) {
    if (keys) keys[i] = f16_bits_to_f32(hk[i]);
    if (values) values[i] = f16_bits_to_f32(hv[i]);
  }
  return NFB_OK;
}

int nfb_kv_synth(nfb_ctx* c, int layer, int count, uint64_t seed) {
  TRY(check_layer(c, layer));
  if (count < 0 || count > c->max_seq) return fail(NFB_EINVAL, "KV synth count out of range");
  cudaSetDevice(c->device);
  LayerBufs& b = c->layers[layer];
  const int H = c->desc.n_heads, d = c->desc.d_head;
  if (count) {
    const int grid = 148 * 8;
    const int h0 = c->tp_rank * H;  // tensor parallel: this rank's heads of the full stream
    kv_synth_kernel<<<grid, 256, 0, c->stream>>>(seed, 0, H, count, d, c->max_seq, b.kc, h0);
    kv_synth_kernel<<<grid, 256, 0, c->stream>>>(seed, 1, H, count, d, c->max_seq, b.vc, h0);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  }
  b.kv_len = count;
  return NFB_OK;
}

static int check_ready(nfb_ctx* c, int l0, int l1, int pos, bool rewind = false) {
  for (int l = l0; l < l1; ++l) {
    const LayerBufs& b = c->layers[l];
    if (!b.weights) return fail(NFB_ESTATE, "weights of layer " + std::to_string(l) + " not set");
    if (b.kv_len != pos && !(rewind && pos <= b.kv_len))
      return fail(NFB_EINVAL, "cache holds " + std::to_string(b.kv_len) + " positions, expected " +
                                  std::to_string(pos));
  }
  if (pos < 0 || pos + 1 > c->max_seq)
    return fail(NFB_EINVAL, "position " + std::to_string(pos) + " exceeds KV capacity " +
                                std::to_string(c->max_seq));
  return NFB_OK;
}

static int check_finite(const float* x, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return fail(NFB_EINVAL, "non-finite activation");
  return NFB_OK;
}

int nfb_block_step(nfb_ctx* c, int layer, int pos, const float* x_in, float* x_out) {
  TRY(check_layer(c, layer));
  if (!x_in || !x_out) return fail(NFB_EINVAL, "null x");
  TRY(check_ready(c, layer, layer + 1, pos));
  TRY(check_finite(x_in, c->desc.hidden));
  cudaSetDevice(c->device);
  const int h = c->desc.hidden;
  memcpy(c->h_x, x_in, (size_t)h * 4);
  c->h_state[0] = pos;
  CK(cudaMemcpyAsync(c->xs, c->h_x, (size_t)h * 4, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->state, c->h_state, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  Params p = base_params(c);
  p.l0 = layer;
  p.l1 = layer + 1;
  p.in_mode = IN_X;
  p.head_mode = HEAD_NONE;
  p.advance_pos = 0;
  TRY(reset_counters(c, c->stream));
  TRY(launch(c, p, c->stream));
  CK(cudaMemcpyAsync(c->h_hidden, c->xs + h, (size_t)h * 4, cudaMemcpyDeviceToHost, c->stream));
  TRY(check_device_error(c));
  memcpy(x_out, c->h_hidden, (size_t)h * 4);
  c->layers[layer].kv_len = pos + 1;
  c->decode_pos = -1;
  return NFB_OK;
}

int nfb_forward(nfb_ctx* c, int pos, const float* x_in, float* hidden_out, float* logits_out,
                int head_mode) {
  if (!c || !x_in) return fail(NFB_EINVAL, "null argument");
  if (c->tp_size > 1)
    return fail(NFB_EUNSUPPORTED, "tensor-parallel contexts: use nfb_block_step per layer or the decode API");
  const int L = c->desc.n_layers, h = c->desc.hidden, V = c->desc.vocab;
  TRY(check_ready(c, 0, L, pos));
  TRY(check_finite(x_in, h));
  if (head_mode < NFB_HEAD_NONE || head_mode > NFB_HEAD_LM) return fail(NFB_EINVAL, "bad head_mode");
  if (head_mode != NFB_HEAD_NONE && !c->has_unembed) return fail(NFB_ESTATE, "unembedding not set");
  if (head_mode == NFB_HEAD_LM && !c->has_lnf) return fail(NFB_ESTATE, "final LN not set");
  cudaSetDevice(c->device);
  memcpy(c->h_x, x_in, (size_t)h * 4);
  c->h_state[0] = pos;
  CK(cudaMemcpyAsync(c->xs, c->h_x, (size_t)h * 4, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->state, c->h_state, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  Params p = base_params(c);
  p.l0 = 0;
  p.l1 = L;
  p.in_mode = IN_X;
  p.head_mode = head_mode;
  p.advance_pos = 0;
  TRY(reset_counters(c, c->stream));
  TRY(launch(c, p, c->stream));
  if (hidden_out)
    CK(cudaMemcpyAsync(c->h_hidden, c->xs, (size_t)(L + 1) * h * 4, cudaMemcpyDeviceToHost, c->stream));
  if (logits_out && head_mode != NFB_HEAD_NONE)
    CK(cudaMemcpyAsync(c->h_logits, c->logits, (size_t)V * 4, cudaMemcpyDeviceToHost, c->stream));
  TRY(check_device_error(c));
  if (hidden_out) memcpy(hidden_out, c->h_hidden, (size_t)(L + 1) * h * 4);
  if (logits_out && head_mode != NFB_HEAD_NONE) memcpy(logits_out, c->h_logits, (size_t)V * 4);
  for (int l = 0; l < L; ++l) c->layers[l].kv_len = pos + 1;
  c->decode_pos = -1;
  return NFB_OK;
}

// ---- device-resident variants (torch CUDA tensors: raw pointer + stream) ----
int nfb_block_step_dev(nfb_ctx* c, int layer, int pos, const float* x_in, float* x_out, void* stream) {
  TRY(check_layer(c, layer));
  if (!x_in || !x_out) return fail(NFB_EINVAL, "null x");
  TRY(check_ready(c, layer, layer + 1, pos));
  cudaSetDevice(c->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  const int h = c->desc.hidden;
  CK(cudaMemcpyAsync(c->xs, x_in, (size_t)h * 4, cudaMemcpyDeviceToDevice, st));
  set_pos_kernel<<<1, 1, 0, st>>>(c->state, pos);
  CK(cudaGetLastError());
  Params p = base_params(c);
  p.l0 = layer;
  p.l1 = layer + 1;
  p.in_mode = IN_X;
  p.head_mode = HEAD_NONE;
  p.advance_pos = 0;
  TRY(reset_counters(c, st));
  TRY(launch(c, p, st));
  CK(cudaMemcpyAsync(x_out, c->xs + h, (size_t)h * 4, cudaMemcpyDeviceToDevice, st));
  c->layers[layer].kv_len = pos + 1;
  c->decode_pos = -1;
  return NFB_OK;
}

int nfb_forward_dev(nfb_ctx* c, int pos, const float* x_in, float* hidden_out, float* logits_out, int head_mode,
                    void* stream) {
  if (!c || !x_in) return fail(NFB_EINVAL, "null argument");
  if (c->tp_size > 1)
    return fail(NFB_EUNSUPPORTED, "tensor-parallel contexts: use nfb_block_step per layer or the decode API");
  const int L = c->desc.n_layers, h = c->desc.hidden, V = c->desc.vocab;
  TRY(check_ready(c, 0, L, pos));
  if (head_mode < NFB_HEAD_NONE || head_mode > NFB_HEAD_LM) return fail(NFB_EINVAL, "bad head_mode");
  if (head_mode != NFB_HEAD_NONE && !c->has_unembed) return fail(NFB_ESTATE, "unembedding not set");
  if (head_mode == NFB_HEAD_LM && !c->has_lnf) return fail(NFB_ESTATE, "final LN not set");
  cudaSetDevice(c->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  CK(cudaMemcpyAsync(c->xs, x_in, (size_t)h * 4, cudaMemcpyDeviceToDevice, st));
  set_pos_kernel<<<1, 1, 0, st>>>(c->state, pos);
  CK(cudaGetLastError());
  Params p = base_params(c);
  p.l0 = 0;
  p.l1 = L;
  p.in_mode = IN_X;
  p.head_mode = head_mode;
  p.advance_pos = 0;
  TRY(reset_counters(c, st));
  TRY(launch(c, p, st));
  if (hidden_out) CK(cudaMemcpyAsync(hidden_out, c->xs, (size_t)(L + 1) * h * 4, cudaMemcpyDeviceToDevice, st));
  if (logits_out && head_mode != NFB_HEAD_NONE)
    CK(cudaMemcpyAsync(logits_out, c->logits, (size_t)V * 4, cudaMemcpyDeviceToDevice, st));
  for (int l = 0; l < L; ++l) c->layers[l].kv_len = pos + 1;
  c->decode_pos = -1;
  return NFB_OK;
}

int nfb_begin_decode(nfb_ctx* c, int pos, int token) {
  if (!c) return fail(NFB_EINVAL, "null context");
  const int L = c->desc.n_layers;
  TRY(check_ready(c, 0, L, pos, true));  // may rewind: positions >= pos are discarded
  if (!c->has_embed || !c->has_unembed || !c->has_lnf) return fail(NFB_ESTATE, "embedding / LM head not set");
  if (token < 0 || token >= c->full.vocab) return fail(NFB_EINVAL, "token out of range");
  cudaSetDevice(c->device);
  CK(cudaStreamSynchronize(c->stream));
  int st[2] = {pos, 0};
  CK(cudaMemcpy(c->state, st, sizeof(st), cudaMemcpyHostToDevice));
  unsigned long long am[2] = {0ull, (0xffffffffull << 32) | (unsigned long long)(0xffffffffu - (uint32_t)token)};
  CK(cudaMemcpy(c->amax, am, sizeof(am), cudaMemcpyHostToDevice));
  TRY(reset_counters(c, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->decode_pos = pos;
  c->decode_step = 0;
  for (auto& b : c->layers) b.kv_len = pos;
  return NFB_OK;
}

static Params decode_params(nfb_ctx* c) {
  Params p = base_params(c);
  p.l0 = 0;
  p.l1 = c->desc.n_layers;
  p.in_mode = IN_TOKEN;
  p.head_mode = HEAD_LM;
  p.advance_pos = 1;
  return p;
}

static int advance_host(nfb_ctx* c, int n) {
  if (c->decode_pos < 0) return fail(NFB_ESTATE, "call nfb_begin_decode first");
  if (c->tp_size > 1 && !c->nccl) return fail(NFB_ESTATE, "tensor-parallel context: call nfb_tp_init first");
  if (c->decode_pos + n > c->max_seq) return fail(NFB_EINVAL, "decode would exceed the KV capacity");
  return NFB_OK;
}

int nfb_decode_step(nfb_ctx* c, void* stream) {
  if (!c) return fail(NFB_EINVAL, "null context");
  TRY(advance_host(c, 1));
  cudaSetDevice(c->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  if (c->nccl) TRY(tp_token(c, st));  // tensor parallel (incl. a 1-rank communicator)
  else TRY(launch(c, decode_params(c), st));
  c->decode_pos += 1;
  c->decode_step += 1;
  for (auto& b : c->layers) b.kv_len = c->decode_pos;
  return NFB_OK;
}

int nfb_graph_capture(nfb_ctx* c) {
  if (!c) return fail(NFB_EINVAL, "null context");
  cudaSetDevice(c->device);
  if (c->gexec) {
    cudaGraphExecDestroy(c->gexec);
    c->gexec = nullptr;
  }
  for (auto& gt : c->gtok)
    if (gt) {
      cudaGraphExecDestroy(gt);
      gt = nullptr;
    }
  if (c->graph) {
    cudaGraphDestroy(c->graph);
    c->graph = nullptr;
  }
  // Resolve the cooperative fallback outside capture (a refused launch would
  // invalidate the capture).
  CK(cudaStreamSynchronize(c->stream));
  if (c->nccl) {
    // resolve the cooperative-launch fallback eagerly: one launch of layer 0
    // as a plain block step is not needed -- tp_token's launch() handles it,
    // so just capture the whole token sequence
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int r = tp_token(c, c->stream);
    cudaGraph_t g = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(c->stream, &g);
    if (r != NFB_OK) {
      if (g) cudaGraphDestroy(g);
      return r;
    }
    if (e2 != cudaSuccess) return fail(NFB_ECUDA, std::string("end capture: ") + cudaGetErrorString(e2));
    c->graph = g;
    CK(cudaGraphInstantiate(&c->gexec, g, 0));
    return NFB_OK;
  }
  const Params p = decode_params(c);
  const int variant = kernel_variant(c);
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t e = launch_decode(p, variant, c->grid, c->block, c->smem, c->stream, c->coop);
  cudaGraph_t g = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(c->stream, &g);
  if ((e != cudaSuccess || e2 != cudaSuccess) && c->coop) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    c->coop = false;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    e = launch_decode(p, variant, c->grid, c->block, c->smem, c->stream, false);
    e2 = cudaStreamEndCapture(c->stream, &g);
  }
  if (e != cudaSuccess) return fail(NFB_ECUDA, std::string("capture launch: ") + cudaGetErrorString(e));
  if (e2 != cudaSuccess) return fail(NFB_ECUDA, std::string("end capture: ") + cudaGetErrorString(e2));
  c->graph = g;
  CK(cudaGraphInstantiate(&c->gexec, g, 0));
  // the serving-step graphs (nfb_step_token): token in -> decode -> token out
  for (int par = 0; par < 2; ++par) {
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    cudaMemcpyAsync(c->amax + (par ^ 1), c->h_tok, 8, cudaMemcpyHostToDevice, c->stream);
    e = launch_decode(p, variant, c->grid, c->block, c->smem, c->stream, c->coop);
    cudaMemcpyAsync(c->h_tok + 1, c->amax + par, 8, cudaMemcpyDeviceToHost, c->stream);
    cudaGraph_t gt = nullptr;
    e2 = cudaStreamEndCapture(c->stream, &gt);
    if (e != cudaSuccess || e2 != cudaSuccess) {
      if (gt) cudaGraphDestroy(gt);
      return fail(NFB_ECUDA, std::string("step graph capture: ") + cudaGetErrorString(e != cudaSuccess ? e : e2));
    }
    const cudaError_t ei = cudaGraphInstantiate(&c->gtok[par], gt, 0);
    cudaGraphDestroy(gt);
    if (ei != cudaSuccess) return fail(NFB_ECUDA, std::string("step graph instantiate: ") + cudaGetErrorString(ei));
  }
  return NFB_OK;
}

int nfb_graph_replay(nfb_ctx* c, int n, void* stream) {
  if (!c) return fail(NFB_EINVAL, "null context");
  if (!c->gexec) return fail(NFB_ESTATE, "call nfb_graph_capture first");
  if (n < 0) return fail(NFB_EINVAL, "n must be >= 0");
  TRY(advance_host(c, n));
  cudaSetDevice(c->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  for (int i = 0; i < n; ++i) CK(cudaGraphLaunch(c->gexec, st));
  c->decode_pos += n;
  c->decode_step += n;
  for (auto& b : c->layers) b.kv_len = c->decode_pos;
  return NFB_OK;
}

int nfb_step_token(nfb_ctx* c, int token, int* next_token) {
  if (!c || !next_token) return fail(NFB_EINVAL, "null argument");
  if (token < 0 || token >= c->full.vocab) return fail(NFB_EINVAL, "token out of range");
  TRY(advance_host(c, 1));
  cudaSetDevice(c->device);
  const int par = c->decode_step & 1;
  // the step reads its input token from slot par^1 and writes its argmax to slot par
  c->h_tok[0] = (0xffffffffull << 32) | (unsigned long long)(0xffffffffu - (uint32_t)token);
  if (c->gtok[par]) {
    CK(cudaGraphLaunch(c->gtok[par], c->stream));  // H2D + decode + D2H in one launch
  } else {
    CK(cudaMemcpyAsync(c->amax + (par ^ 1), c->h_tok, 8, cudaMemcpyHostToDevice, c->stream));
    if (c->gexec) {
      CK(cudaGraphLaunch(c->gexec, c->stream));
    } else if (c->nccl) {
      TRY(tp_token(c, c->stream));
    } else {
      TRY(launch(c, decode_params(c), c->stream));
    }
    CK(cudaMemcpyAsync(c->h_tok + 1, c->amax + par, 8, cudaMemcpyDeviceToHost, c->stream));
  }
  TRY(check_device_error(c));
  c->decode_pos += 1;
  c->decode_step += 1;
  for (auto& b : c->layers) b.kv_len = c->decode_pos;
  *next_token = (int)(0xffffffffu - (uint32_t)(c->h_tok[1] & 0xffffffffull));
  return NFB_OK;
}

int nfb_set_option(nfb_ctx* c, int option, int value) {
  if (!c) return fail(NFB_EINVAL, "null context");
  cudaSetDevice(c->device);
  if (option == NFB_OPT_TRACE) {
    if (value && !c->trace) {
      c->trace_stride = kTraceHeader + kTracePerLayer * c->desc.n_layers + kTraceStageWords;
      TRY(dalloc(c, &c->trace, (size_t)c->grid * c->trace_stride));
    } else if (!value) {
      c->trace = nullptr;  // buffer stays in allocs until destroy
    }
  } else if (option == NFB_OPT_DYNAMIC_MLP) {
    c->dyn_mlp = value ? 1 : 0;
  } else if (option == NFB_OPT_HEAD_WEIGHT) {
    if (value < 0 || value > 1000) return fail(NFB_EINVAL, "head weight must be in [0, 1000] percent");
    c->head_weight_pct = value;
  } else if (option == NFB_OPT_ASSIST) {
    const int C = c->C, d3 = 3 * c->desc.d_head;
    if (value && (value > 6 || d3 % (C + value) || (d3 / (C + value)) % 4 || c->grid <= C * std::min(c->desc.n_heads, c->n_clusters)))
      return fail(NFB_EUNSUPPORTED, "QKV assist needs CTAs without heads and parts of a multiple of 4 rows");
    c->assist = value;
  } else if (option == NFB_OPT_DETERMINISTIC) {
    c->deterministic = value ? 1 : 0;
  } else if (option == NFB_OPT_PREFETCH_KB) {
    if (value < 0 || value > 65536) return fail(NFB_EINVAL, "prefetch lead must be in [0, 65536] KiB");
    c->pf_ahead = value * 1024;
  } else {
    return fail(NFB_EINVAL, "unknown option");
  }
  if (c->gexec) {  // captured params are stale
    cudaGraphExecDestroy(c->gexec);
    c->gexec = nullptr;
  }
  for (auto& gt : c->gtok)
    if (gt) {
      cudaGraphExecDestroy(gt);
      gt = nullptr;
    }
  return NFB_OK;
}

int nfb_read_trace(nfb_ctx* c, unsigned long long* out, int n) {
  if (!c || !out) return fail(NFB_EINVAL, "null argument");
  if (!c->trace) return fail(NFB_ESTATE, "tracing not enabled");
  TRY(nfb_sync(c));
  const size_t total = (size_t)c->grid * c->trace_stride;
  CK(cudaMemcpy(out, c->trace, std::min<size_t>(total, (size_t)n) * 8, cudaMemcpyDeviceToHost));
  return NFB_OK;
}

int nfb_sync(nfb_ctx* c) {
  if (!c) return fail(NFB_EINVAL, "null context");
  cudaSetDevice(c->device);
  return check_device_error(c);
}

int nfb_get_state(nfb_ctx* c, int* pos, int* step) {
  if (!c) return fail(NFB_EINVAL, "null context");
  TRY(nfb_sync(c));
  int st[2];
  CK(cudaMemcpy(st, c->state, sizeof(st), cudaMemcpyDeviceToHost));
  if (pos) *pos = st[0];
  if (step) *step = st[1];
  return NFB_OK;
}

int nfb_read_tokens(nfb_ctx* c, int* tokens, int n, int* last_argmax) {
  if (!c) return fail(NFB_EINVAL, "null context");
  if (n < 0 || n > c->max_seq) return fail(NFB_EINVAL, "n out of range");
  TRY(nfb_sync(c));
  if (tokens && n) CK(cudaMemcpy(tokens, c->tokens, (size_t)n * sizeof(int), cudaMemcpyDeviceToHost));
  if (last_argmax) {
    int st[2];
    CK(cudaMemcpy(st, c->state, sizeof(st), cudaMemcpyDeviceToHost));
    unsigned long long am[2];
    CK(cudaMemcpy(am, c->amax, sizeof(am), cudaMemcpyDeviceToHost));
    const unsigned long long v = am[(st[1] + 1) & 1];  // written by step st[1]-1
    *last_argmax = (int)(0xffffffffu - (uint32_t)(v & 0xffffffffull));
  }
  return NFB_OK;
}

int nfb_read_hidden(nfb_ctx* c, float* out) {
  if (!c || !out) return fail(NFB_EINVAL, "null argument");
  TRY(nfb_sync(c));
  CK(cudaMemcpy(out, c->xs, (size_t)(c->desc.n_layers + 1) * c->desc.hidden * 4, cudaMemcpyDeviceToHost));
  return NFB_OK;
}

int nfb_read_logits(nfb_ctx* c, float* out) {
  if (!c || !out) return fail(NFB_EINVAL, "null argument");
  TRY(nfb_sync(c));
  CK(cudaMemcpy(out, c->logits, (size_t)c->desc.vocab * 4, cudaMemcpyDeviceToHost));
  return NFB_OK;
}


int nfb_create_tp(const nfb_model_desc* full, int device, int max_seq, int cluster_size, int max_clusters,
                  int tp_rank, int tp_size, nfb_ctx** out) {
  if (!full || !out) return fail(NFB_EINVAL, "null argument");
  if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size) return fail(NFB_EINVAL, "bad tensor-parallel rank / size");
  if (full->n_heads % tp_size || full->d_mlp % tp_size || full->vocab % tp_size)
    return fail(NFB_EUNSUPPORTED, "n_heads, d_mlp and vocab must divide by the tensor-parallel size");
  if (tp_size > 1 && !full->parallel_residual)
    return fail(NFB_EUNSUPPORTED, "tensor parallelism needs the parallel residual (one all-reduce per layer)");
  nfb_model_desc m = *full;
  m.n_heads /= tp_size;
  m.d_mlp /= tp_size;
  m.vocab /= tp_size;
  const int r = create_ctx(&m, full, device, max_seq, cluster_size, max_clusters, out);
  if (r != NFB_OK) return r;
  (*out)->tp_rank = tp_rank;
  (*out)->tp_size = tp_size;
  return NFB_OK;
}

int nfb_tp_unique_id(void* out128) {
  if (!out128) return fail(NFB_EINVAL, "null argument");
  NcclApi& n = nccl_api();
  if (!n.ok) return fail(NFB_EUNSUPPORTED, "libnccl.so.2 not found");
  ncclUniqueId id;
  NCK(n.getUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
  return NFB_OK;
}

int nfb_tp_init(nfb_ctx* c, const void* unique_id128) {
  if (!c || !unique_id128) return fail(NFB_EINVAL, "null argument");
  NcclApi& n = nccl_api();
  if (!n.ok) return fail(NFB_EUNSUPPORTED, "libnccl.so.2 not found");
  cudaSetDevice(c->device);
  ncclUniqueId id;
  memcpy(&id, unique_id128, sizeof(id));
  ncclComm_t comm = nullptr;
  NCK(n.commInitRank(&comm, c->tp_size, id, c->tp_rank));
  c->nccl = comm;
  return NFB_OK;
}

int nfb_tp_info(nfb_ctx* c, int* tp_rank, int* tp_size) {
  if (!c || !tp_rank || !tp_size) return fail(NFB_EINVAL, "null argument");
  *tp_rank = c->tp_rank;
  *tp_size = c->tp_size;
  return NFB_OK;
}

int nfb_head_logits(nfb_ctx* c, const float* h_in, float* logits_out, int head_mode) {
  if (!c || !h_in || !logits_out) return fail(NFB_EINVAL, "null argument");
  if (head_mode != NFB_HEAD_PROBE && head_mode != NFB_HEAD_LM) return fail(NFB_EINVAL, "bad head_mode");
  if (!c->has_unembed) return fail(NFB_ESTATE, "unembedding not set");
  if (head_mode == NFB_HEAD_LM && !c->has_lnf) return fail(NFB_ESTATE, "final LN not set");
  const int L = c->desc.n_layers, h = c->desc.hidden, V = c->desc.vocab;
  TRY(check_finite(h_in, h));
  cudaSetDevice(c->device);
  memcpy(c->h_x, h_in, (size_t)h * 4);
  CK(cudaMemcpyAsync(c->xs + (size_t)L * h, c->h_x, (size_t)h * 4, cudaMemcpyHostToDevice, c->stream));
  Params p = base_params(c);
  p.l0 = p.l1 = L;
  p.xs = c->xs + (size_t)L * h;
  p.in_mode = IN_X;
  p.head_mode = head_mode;
  p.advance_pos = 0;
  p.state_update = 0;
  TRY(reset_counters(c, c->stream));
  TRY(launch(c, p, c->stream));
  CK(cudaMemcpyAsync(c->h_logits, c->logits, (size_t)V * 4, cudaMemcpyDeviceToHost, c->stream));
  TRY(check_device_error(c));
  memcpy(logits_out, c->h_logits, (size_t)V * 4);
  return NFB_OK;
}


// ===========================================================================
// Batched decode (BASELINE.json configs[3]): see csrc/nfb_batch.cu.
// ===========================================================================
// Y = W . A on the tcgen05 GEMM (csrc/nfb_umma.cu): role j of the current
// plan set (0 qkv, 1 out, 2 up, 3 down, 4 lm).
static int ugemm(nfb_ctx* c, cudaStream_t st, int j, const void* Wb, const void* Ab) {
  const cudaError_t e = umma_gemm(st, c->uplan[j], Wb, Ab, c->uws[j], c->err, true);
  if (e != cudaSuccess) return fail(NFB_ECUDA, std::string("umma_gemm launch: ") + cudaGetErrorString(e));
  return NFB_OK;
}

// (Re)build the blocked weight copies after a weight change, and the GEMM
// plans when the batch size changes.
static int batch_prepare(nfb_ctx* c, cudaStream_t st) {
  const int h = c->desc.hidden, mm = c->desc.d_mlp, L = c->desc.n_layers, V = c->desc.vocab;
  if (c->bt_ver != c->wver) {
    for (int l = 0; l < L; ++l) {
      const LayerBufs& w = c->layers[l];
      __half** bw = reinterpret_cast<__half**>(&c->bw[(size_t)4 * l]);
      umma_block_weights(st, reinterpret_cast<const __half*>(w.wqkv), 3 * h, h, h, false, bw[0]);
      umma_block_weights(st, reinterpret_cast<const __half*>(w.woT), h, h, h, true, bw[1]);    // W_out = woT^T
      umma_block_weights(st, reinterpret_cast<const __half*>(w.wup), mm, h, h, false, bw[2]);
      umma_block_weights(st, reinterpret_cast<const __half*>(w.wdT), h, mm, h, true, bw[3]);   // W_down = wdT^T
    }
    if (c->has_unembed)
      umma_block_weights(st, reinterpret_cast<const __half*>(c->unembed), V, h, h, false,
                         reinterpret_cast<__half*>(c->blm));
    CK(cudaGetLastError());
    c->bt_ver = c->wver;
  }
  if (c->uplan_rows != c->bcur) {
    const int shapes[5][2] = {{3 * h, h}, {h, h}, {mm, h}, {h, mm}, {V, h}};
    // The MLP branch's GEMMs (up, down) run beside the attention branch; at
    // B <= 8 they get one CTA per SM instead of 1.5, leaving the extra slots
    // to the critical attention chain (C4 B = 2 / 3 / 4 / 8: +2.9 / +3.0 /
    // +2.7 / +1.5 %; B = 16: -2.4 %, so larger batches keep 1.5).
    // NFB_UMMA_MLP_SMS overrides (never above the SM count: the partial
    // buffers are sized for it).
    int mlp_sms = c->bcur <= 8 ? (2 * c->sm_count + 2) / 3 : c->sm_count;
    if (const char* e = getenv("NFB_UMMA_MLP_SMS")) mlp_sms = std::max(1, std::min(c->sm_count, atoi(e)));
    for (int j = 0; j < 5; ++j)
      c->uplan[j] = umma_plan(shapes[j][0], 2 * c->bcur, shapes[j][1], (j == 2 || j == 3) ? mlp_sms : c->sm_count);
    c->uplan_rows = c->bcur;
  }
  return NFB_OK;
}

// One token for all bcur sequences: layers (LN -> QKV GEMM -> RoPE/append ->
// split-KV attention -> W_out GEMM, LN2 -> up GEMM -> GELU -> down GEMM ->
// residual) then final LN -> LM GEMM -> argmax.  in_token: x from btok.
// Every launch carries the PDL attribute (launch_pdl / umma_gemm).
static int batch_token(nfb_ctx* c, cudaStream_t st, bool in_token, bool head, bool prefill = false) {
  const nfb_model_desc& m = c->desc;
  const int B = c->bcur, h = m.hidden, H = m.n_heads, d = m.d_head, mm = m.d_mlp, V = m.vocab;
  const int L = m.n_layers, S = c->bsplit;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusNone) TRY(batch_prepare(c, st));
  else if (c->bt_ver != c->wver || c->uplan_rows != c->bcur)
    return fail(NFB_ESTATE, "batched graph capture needs prepared weights / plans (call batch_prepare first)");
  const int np = c->uplan[0].n_pad;
  __half* a1 = reinterpret_cast<__half*>(c->ba1);
  __half* a2 = reinterpret_cast<__half*>(c->ba2);
  __half* actx = reinterpret_cast<__half*>(c->bctx);
  __half* ag = reinterpret_cast<__half*>(c->bg);
  const UOut oq = umma_out(c->uplan[0], c->uws[0]), oz = umma_out(c->uplan[1], c->uws[1]);
  const UOut ou = umma_out(c->uplan[2], c->uws[2]), od = umma_out(c->uplan[3], c->uws[3]);
  if (in_token)
    CK(launch_pdl(embed_kernel, dim3(B), dim3(256), 0, st, c->btok, reinterpret_cast<const __half*>(c->embed), h, V,
                  c->bx));
  const float scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
  for (int l = 0; l < L; ++l) {
    const LayerBufs& w = c->layers[l];
    uint16_t* const* bw = &c->bw[(size_t)4 * l];
    CK(launch_pdl(ln_hilo_kernel, dim3(B), dim3(256), 0, st, c->bx, B, h, (float)m.ln_eps, w.ln1g, w.ln1b, w.ln2g,
                  w.ln2b, a1, a2, np));
    // The MLP branch forks right after the LNs (bfork 4, default: the up GEMM
    // streams beside the QKV GEMM -- both are latency-dominated at small B;
    // C4 B = 2 / 4 / 16: +1.4 / +3 / +0.8 %) or after the QKV GEMM (bfork 1).
    if (c->bfork == 4) CK(cudaEventRecord(c->bev[0], st));
    if (!(c->bskip & 4)) TRY(ugemm(c, st, 0, bw[0], a1));
    // batch: sequence b has its own cache; prefill: the T prompt rows share
    // the context's cache at consecutive positions (causal)
    __half* kc = reinterpret_cast<__half*>(prefill ? w.kc : c->bkc[l]);
    __half* vc = reinterpret_cast<__half*>(prefill ? w.vc : c->bvc[l]);
    const size_t sstride = prefill ? 0 : (size_t)H * c->max_seq * d;
    const int pstep = prefill ? 1 : 0;
    // MLP branch (independent of the attention under the parallel residual)
    cudaStream_t sm = st;
    if (c->bfork) {
      if (c->bfork != 4) CK(cudaEventRecord(c->bev[0], st));
      CK(cudaStreamWaitEvent(c->bstream2, c->bev[0], 0));
      sm = c->bstream2;
    }
    if (!(c->bskip & 1)) {
      if (!(c->bskip & 4)) TRY(ugemm(c, sm, 2, bw[2], a2));
      CK(launch_pdl(gelu_hilo_kernel, dim3(B, (mm + 255) / 256), dim3(256), 0, sm, ou, B, mm, w.bup, m.gelu_exact,
                    ag, np));
      if (!(c->bskip & 4)) TRY(ugemm(c, sm, 3, bw[3], ag));
    }
    if (c->bfork) CK(cudaEventRecord(c->bev[1], sm));
    if (!(c->bskip & 2)) {
      CK(launch_pdl(attn_prep_kernel, dim3(B, H), dim3(128), (size_t)3 * d * 4, st, oq, B, H, d, m.rotary_dims,
                    c->bstate, c->max_seq, w.bqkv, c->rope, c->bq, kc, vc, pstep, sstride));
      if (prefill && c->bprefill_rows)  // one tile fetch per kPrefillRows prompt rows
        CK(launch_pdl(attn_tile_rows_kernel, dim3(H * ((B + attn_prefill_rows() - 1) / attn_prefill_rows()), S),
                      dim3(attn_tile_positions()), attn_tile_rows_smem(d), st, c->bq, kc, vc, B, H, d, c->max_seq,
                      c->bstate, scale_log2, c->bpart));
      else
        CK(launch_pdl(attn_tile_kernel, dim3(B * H, S), dim3(attn_tile_positions()), attn_tile_smem(d), st, c->bq, kc, vc, B, H, d,
                    c->max_seq, c->bstate, scale_log2, c->bpart, pstep, sstride));
      CK(launch_pdl(attn_combine_kernel, dim3(B * H), dim3(128), 0, st, c->bpart, S, B, H, d, actx, np));
      if (!(c->bskip & 4)) TRY(ugemm(c, st, 1, bw[1], actx));
    }
    if (c->bfork) CK(cudaStreamWaitEvent(st, c->bev[1], 0));
    CK(launch_pdl(residual_kernel, dim3(B, (h + 255) / 256), dim3(256), 0, st, c->bx, B, h, oz, w.bo, od, w.bd));
  }
  if (head) {
    CK(launch_pdl(ln_hilo_kernel, dim3(B), dim3(256), 0, st, c->bx, B, h, (float)m.ln_eps, c->lnfg, c->lnfb,
                  (const float*)nullptr, (const float*)nullptr, a1, (__half*)nullptr, np));
    TRY(ugemm(c, st, 4, c->blm, a1));
    CK(launch_pdl(argmax_kernel, dim3(B, 37), dim3(256), 0, st, umma_out(c->uplan[4], c->uws[4]), B, V, c->bamax,
                  c->blogits));
  }
  CK(launch_pdl(advance_kernel, dim3(1), dim3(128), 0, st, c->bstate, head ? c->bamax : (unsigned long long*)nullptr,
                c->btok, B, V));
  return NFB_OK;
}

int nfb_batch_init(nfb_ctx* c, int max_batch) {
  if (!c) return fail(NFB_EINVAL, "null context");
  if (max_batch < 1 || max_batch > 128) return fail(NFB_EINVAL, "max_batch must be in [1, 128] (UMMA N = 2B <= 256)");
  if (c->bmax) return fail(NFB_ESTATE, "batch buffers already allocated");
  if (c->tp_size > 1) return fail(NFB_EUNSUPPORTED, "batched decode is single-GPU");
  if (!c->desc.parallel_residual) return fail(NFB_EUNSUPPORTED, "batched decode needs the parallel residual");
  if (c->desc.d_head > 128) return fail(NFB_EUNSUPPORTED, "batched decode needs d_head <= 128");
  cudaSetDevice(c->device);
  const nfb_model_desc& m = c->desc;
  const size_t B = max_batch, h = m.hidden, H = m.n_heads, d = m.d_head, mm = m.d_mlp, V = m.vocab;
  // KV tiles of 128 positions per (sequence, head) over the whole cache
  // (positions come from device state, so the grid covers max_seq; tiles
  // past the current length exit at once)
  c->bsplit = (c->max_seq + attn_tile_positions() - 1) / attn_tile_positions();
  if (c->bsplit > 256) return fail(NFB_EUNSUPPORTED, "batched decode needs max_seq <= 32768");
  {
    const cudaError_t e2 = cudaFuncSetAttribute(attn_tile_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)attn_tile_rows_smem((int)d));
    if (e2 != cudaSuccess) return fail(NFB_ECUDA, std::string("attn_tile_rows smem attribute: ") + cudaGetErrorString(e2));
  }
  {
    const cudaError_t e = cudaFuncSetAttribute(attn_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)attn_tile_smem((int)d));
    if (e != cudaSuccess) return fail(NFB_ECUDA, std::string("attn_tile smem attribute: ") + cudaGetErrorString(e));
  }
  c->bkc.resize(m.n_layers);
  c->bvc.resize(m.n_layers);
  c->bw.resize((size_t)4 * m.n_layers);
  int r = NFB_OK;
  const int shapes[5][2] = {{3 * (int)h, (int)h}, {(int)h, (int)h}, {(int)mm, (int)h}, {(int)h, (int)mm}, {(int)V, (int)h}};
  for (int l = 0; l < m.n_layers; ++l)
    for (int j = 0; j < 4; ++j)
      if ((r = dalloc(c, &c->bw[(size_t)4 * l + j], umma_blocked_elems(shapes[j][0], shapes[j][1])))) return r;
  if ((r = dalloc(c, &c->blm, umma_blocked_elems((int)V, (int)h)))) return r;
  c->bt_ver = 0;
  for (int l = 0; l < m.n_layers; ++l)
    if ((r = dalloc(c, &c->bkc[l], B * H * c->max_seq * d)) || (r = dalloc(c, &c->bvc[l], B * H * c->max_seq * d)))
      return r;
  const int npm = (2 * (int)B + 7) / 8 * 8;  // n_pad of the largest batch
  if ((r = dalloc(c, &c->bx, B * h)) || (r = dalloc(c, &c->bq, B * h)) ||
      (r = dalloc(c, &c->bpart, B * H * c->bsplit * (d + 2))) || (r = dalloc(c, &c->blogits, B * V)) ||
      (r = dalloc(c, &c->ba1, umma_act_elems(npm, (int)h))) || (r = dalloc(c, &c->ba2, umma_act_elems(npm, (int)h))) ||
      (r = dalloc(c, &c->bctx, umma_act_elems(npm, (int)h))) || (r = dalloc(c, &c->bg, umma_act_elems(npm, (int)mm))) ||
      (r = dalloc(c, &c->btok, B)) || (r = dalloc(c, &c->bstate, 4)) || (r = dalloc(c, &c->bamax, B)))
    return r;
  CK(cudaStreamCreateWithFlags(&c->bstream2, cudaStreamNonBlocking));
  for (auto& e : c->bev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (getenv("NFB_BATCH_FORK")) c->bfork = atoi(getenv("NFB_BATCH_FORK"));
  if (getenv("NFB_BATCH_SKIP")) c->bskip = atoi(getenv("NFB_BATCH_SKIP"));
  if (getenv("NFB_PREFILL_ROWS")) c->bprefill_rows = atoi(getenv("NFB_PREFILL_ROWS"));
  // stream-K partials per role: tiles x pieces x n_pad x 128 (pieces depend
  // on M, K and the grid only; n_pad is largest at the largest batch)
  for (int j = 0; j < 5; ++j)
    if ((r = dalloc(c, &c->uws[j], umma_plan(shapes[j][0], 2 * (int)B, shapes[j][1], c->sm_count).ws_floats())))
      return r;
  c->uplan_rows = 0;
  c->bmax = max_batch;
  return NFB_OK;
}

int nfb_batch_kv_synth(nfb_ctx* c, int count, uint64_t base_seed) {
  if (!c) return fail(NFB_EINVAL, "null context");
  if (!c->bmax) return fail(NFB_ESTATE, "call nfb_batch_init first");
  if (count < 0 || count > c->max_seq) return fail(NFB_EINVAL, "KV synth count out of range");
  cudaSetDevice(c->device);
  const int H = c->desc.n_heads, d = c->desc.d_head;
  for (int l = 0; l < c->desc.n_layers; ++l) {
    // layer l: all bmax sequences as one stream of bmax * H heads (seed kv_seed(base, l))
    const uint64_t seed = base_seed + 0x10000 + l;
    if (count) {
      kv_synth_kernel<<<148 * 8, 256, 0, c->stream>>>(seed, 0, H * c->bmax, count, d, c->max_seq, c->bkc[l]);
      kv_synth_kernel<<<148 * 8, 256, 0, c->stream>>>(seed, 1, H * c->bmax, count, d, c->max_seq, c->bvc[l]);
    }
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  return NFB_OK;
}

int nfb_batch_kv_write(nfb_ctx* c, int layer, int seq, int start, int count, const void* keys, const void* values,
                       int dtype) {
  TRY(check_layer(c, layer));
  if (!c->bmax) return fail(NFB_ESTATE, "call nfb_batch_init first");
  if (seq < 0 || seq >= c->bmax || start < 0 || count < 0 || start + count > c->max_seq)
    return fail(NFB_EINVAL, "batch KV write range invalid");
  if (count && (!keys || !values)) return fail(NFB_EINVAL, "null keys/values");
  cudaSetDevice(c->device);
  CK(cudaStreamSynchronize(c->stream));
  const size_t H = c->desc.n_heads, d = c->desc.d_head;
  if (count) {
    std::vector<uint16_t> hk, hv;
    TRY(to_f16_host(keys, dtype, H * count * d, hk));
    TRY(to_f16_host(values, dtype, H * count * d, hv));
    const size_t off = ((size_t)seq * H * c->max_seq + start) * d;
    CK(cudaMemcpy2D(c->bkc[layer] + off, c->max_seq * d * 2, hk.data(), (size_t)count * d * 2, (size_t)count * d * 2,
                    H, cudaMemcpyHostToDevice));
    CK(cudaMemcpy2D(c->bvc[layer] + off, c->max_seq * d * 2, hv.data(), (size_t)count * d * 2, (size_t)count * d * 2,
                    H, cudaMemcpyHostToDevice));
  }
  return NFB_OK;
}

static int batch_setup(nfb_ctx* c, int batch, int pos) {
  if (!c) return fail(NFB_EINVAL, "null context");
  if (!c->bmax) return fail(NFB_ESTATE, "call nfb_batch_init first");
  if (batch < 1 || batch > c->bmax) return fail(NFB_EINVAL, "batch out of range");
  if (pos < 0 || pos >= c->max_seq) return fail(NFB_EINVAL, "position out of range");
  for (int l = 0; l < c->desc.n_layers; ++l)
    if (!c->layers[l].weights) return fail(NFB_ESTATE, "weights of layer " + std::to_string(l) + " not set");
  if (batch != c->bcur && c->bgexec) {
    cudaGraphExecDestroy(c->bgexec);
    c->bgexec = nullptr;
  }
  c->bcur = batch;
  cudaSetDevice(c->device);
  CK(cudaStreamSynchronize(c->stream));
  int st[4] = {pos, 0, 0, 0};
  CK(cudaMemcpy(c->bstate, st, sizeof(st), cudaMemcpyHostToDevice));
  c->bpos = pos;
  return NFB_OK;
}

int nfb_batch_forward(nfb_ctx* c, int batch, int pos, const float* x_in, float* x_out, float* logits_out) {
  TRY(batch_setup(c, batch, pos));
  if (!x_in) return fail(NFB_EINVAL, "null x");
  if (logits_out && (!c->has_unembed || !c->has_lnf)) return fail(NFB_ESTATE, "LM head not set");
  const size_t h = c->desc.hidden;
  CK(cudaMemcpyAsync(c->bx, x_in, (size_t)batch * h * 4, cudaMemcpyHostToDevice, c->stream));
  TRY(batch_token(c, c->stream, false, logits_out != nullptr));
  if (x_out) CK(cudaMemcpyAsync(x_out, c->bx, (size_t)batch * h * 4, cudaMemcpyDeviceToHost, c->stream));
  if (logits_out)
    CK(cudaMemcpyAsync(logits_out, c->blogits, (size_t)batch * c->desc.vocab * 4, cudaMemcpyDeviceToHost, c->stream));
  TRY(check_device_error(c));
  c->bpos = pos + 1;
  return NFB_OK;
}

int nfb_batch_begin(nfb_ctx* c, int batch, int pos, const int* tokens) {
  TRY(batch_setup(c, batch, pos));
  if (!tokens) return fail(NFB_EINVAL, "null tokens");
  if (!c->has_embed || !c->has_unembed || !c->has_lnf) return fail(NFB_ESTATE, "embedding / LM head not set");
  for (int b = 0; b < batch; ++b)
    if (tokens[b] < 0 || tokens[b] >= c->full.vocab) return fail(NFB_EINVAL, "token out of range");
  CK(cudaMemcpy(c->btok, tokens, (size_t)batch * 4, cudaMemcpyHostToDevice));
  return NFB_OK;
}

int nfb_batch_step(nfb_ctx* c, int n, void* stream) {
  if (!c) return fail(NFB_EINVAL, "null context");
  if (!c->bcur || c->bpos < 0) return fail(NFB_ESTATE, "call nfb_batch_begin first");
  if (n < 0 || c->bpos + n > c->max_seq) return fail(NFB_EINVAL, "batch decode would exceed the KV capacity");
  cudaSetDevice(c->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  if (c->bgexec) TRY(batch_prepare(c, st));  // the graph reads the copies in place
  for (int i = 0; i < n; ++i) {
    if (c->bgexec) CK(cudaGraphLaunch(c->bgexec, st));
    else TRY(batch_token(c, st, true, true));
  }
  c->bpos += n;
  return NFB_OK;
}

int nfb_batch_graph_capture(nfb_ctx* c) {
  if (!c) return fail(NFB_EINVAL, "null context");
  if (!c->bcur) return fail(NFB_ESTATE, "call nfb_batch_begin first");
  cudaSetDevice(c->device);
  CK(cudaStreamSynchronize(c->stream));
  if (c->bgexec) {
    cudaGraphExecDestroy(c->bgexec);
    c->bgexec = nullptr;
  }
  if (c->bgraph) {
    cudaGraphDestroy(c->bgraph);
    c->bgraph = nullptr;
  }
  TRY(batch_prepare(c, c->stream));
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  const int r = batch_token(c, c->stream, true, true);
  cudaGraph_t g = nullptr;
  const cudaError_t e2 = cudaStreamEndCapture(c->stream, &g);
  if (r != NFB_OK) {
    if (g) cudaGraphDestroy(g);
    return r;
  }
  if (e2 != cudaSuccess) return fail(NFB_ECUDA, std::string("end capture: ") + cudaGetErrorString(e2));
  c->bgraph = g;
  CK(cudaGraphInstantiate(&c->bgexec, g, 0));
  return NFB_OK;
}

int nfb_batch_read_tokens(nfb_ctx* c, int* tokens) {
  if (!c || !tokens) return fail(NFB_EINVAL, "null argument");
  if (!c->bcur) return fail(NFB_ESTATE, "call nfb_batch_begin first");
  TRY(nfb_sync(c));
  CK(cudaMemcpy(tokens, c->btok, (size_t)c->bcur * 4, cudaMemcpyDeviceToHost));
  return NFB_OK;
}


int nfb_prefill(nfb_ctx* c, int pos, int count, const float* x_in, float* x_out) {
  if (!c || (count && !x_in)) return fail(NFB_EINVAL, "null argument");
  if (!c->bmax) return fail(NFB_ESTATE, "call nfb_batch_init first (prefill runs in chunks of max_batch rows)");
  if (count < 0 || pos < 0 || pos + count > c->max_seq) return fail(NFB_EINVAL, "prefill range invalid");
  for (auto& b : c->layers)
    if (b.kv_len != pos)
      return fail(NFB_EINVAL, "cache holds " + std::to_string(b.kv_len) + " positions, expected " + std::to_string(pos));
  const size_t h = c->desc.hidden;
  TRY(check_finite(x_in, (int)(count * h)));
  cudaSetDevice(c->device);
  for (int t0 = 0; t0 < count; t0 += c->bmax) {
    const int T = std::min(c->bmax, count - t0);
    if (c->bgexec && T != c->bcur) {
      cudaGraphExecDestroy(c->bgexec);
      c->bgexec = nullptr;
    }
    c->bcur = T;
    int st[4] = {pos + t0, 0, 0, 0};
    CK(cudaMemcpyAsync(c->bstate, st, sizeof(st), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->bx, x_in + (size_t)t0 * h, (size_t)T * h * 4, cudaMemcpyHostToDevice, c->stream));
    TRY(batch_token(c, c->stream, false, false, true));
    if (x_out) CK(cudaMemcpyAsync(x_out + (size_t)t0 * h, c->bx, (size_t)T * h * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  TRY(check_device_error(c));
  for (auto& b : c->layers) b.kv_len = pos + count;
  c->decode_pos = -1;
  return NFB_OK;
}

// ---------------------------------------------------------------------------
// Unit-level helpers of the reference's cluster simulator (csrc/nfb_split.cu):
// host float64 arrays in and out, device scratch per call, synchronous on the
// current device's legacy stream.
}  // extern "C"

namespace {
struct DevScratch {
  std::vector<void*> ptrs;
  ~DevScratch() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  cudaError_t get(T** p, size_t bytes) {
    void* q = nullptr;
    const cudaError_t e = cudaMalloc(&q, bytes ? bytes : 8);
    if (e == cudaSuccess) ptrs.push_back(q);
    *p = static_cast<T*>(q);
    return e;
  }
};
}  // namespace

extern "C" {

int nfb_attend_split(const double* q, const double* keys, const double* values, int seq_len, int d, int n_blocks,
                     int merge, uint64_t seed, double scale, double* out) {
  if (!q || !keys || !values || !out) return fail(NFB_EINVAL, "null argument");
  if (seq_len < 1) return fail(NFB_EINVAL, "attention over empty cache");
  if (d < 1 || n_blocks < 1) return fail(NFB_EINVAL, "d and n_blocks must be >= 1");
  if (merge < NFB_MERGE_EXACT || merge > NFB_MERGE_PERMUTED) return fail(NFB_EINVAL, "unknown merge order");
  if (merge == NFB_MERGE_TREE && (n_blocks & (n_blocks - 1)))
    return fail(NFB_EINVAL, "tree merge needs a power-of-two n_blocks");
  const size_t kv = (size_t)seq_len * d * sizeof(double);
  DevScratch s;
  double *dq, *dk, *dv, *lg, *st, *o;
  int* ord;
  void* sc;
  CK(s.get(&dq, d * sizeof(double)));
  CK(s.get(&dk, kv));
  CK(s.get(&dv, kv));
  CK(s.get(&lg, seq_len * sizeof(double)));
  CK(s.get(&st, (size_t)n_blocks * (d + 2) * sizeof(double)));
  CK(s.get(&o, d * sizeof(double)));
  CK(s.get(&ord, n_blocks * sizeof(int)));
  CK(s.get(&sc, attend_split_scratch_bytes(n_blocks, d)));
  CK(cudaMemcpy(dq, q, d * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk, keys, kv, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, values, kv, cudaMemcpyHostToDevice));
  const int mode = n_blocks == 1 ? 4 : merge;
  CK(launch_attend_split(dq, dk, dv, seq_len, d, n_blocks, mode, seed, scale, lg, st, ord, sc, o, nullptr));
  CK(cudaMemcpy(out, o, d * sizeof(double), cudaMemcpyDeviceToHost));
  return NFB_OK;
}

// Float64 golden block on the GPU (csrc/nfb_golden.cu): shape checks, weight
// upload and work buffers for a cache of S positions.
static int golden_setup(const nfb_model_desc* m, const nfb_block_weights* w, int S, DevScratch& s, GoldenBufs& B) {
  const int h = m->hidden, H = m->n_heads, d = m->d_head, mm = m->d_mlp, V = m->vocab, rd = m->rotary_dims;
  if (h < 1 || H < 1 || d < 1 || mm < 1 || V < 1 || H * d != h) return fail(NFB_EINVAL, "invalid model shape");
  if (rd < 2 || rd % 2 || rd > d) return fail(NFB_EINVAL, "rotary_dims must be an even number >= 2 and <= d_head");
  const size_t D = sizeof(double);
  double* wbuf[12];
  const size_t sizes[12] = {(size_t)h, (size_t)h, (size_t)3 * h * h, (size_t)3 * h, (size_t)h * h, (size_t)h,
                            (size_t)h, (size_t)h, (size_t)mm * h, (size_t)mm, (size_t)h * mm, (size_t)h};
  const void* src[12] = {w->ln1_gain, w->ln1_bias, w->qkv_weight, w->qkv_bias, w->out_weight, w->out_bias,
                         w->ln2_gain, w->ln2_bias, w->up_weight, w->up_bias, w->down_weight, w->down_bias};
  for (int i = 0; i < 12; ++i) {
    if (!src[i]) return fail(NFB_EINVAL, "null weight tensor");
    CK(s.get(&wbuf[i], sizes[i] * D));
    CK(cudaMemcpy(wbuf[i], src[i], sizes[i] * D, cudaMemcpyHostToDevice));
  }
  B.ln1g = wbuf[0]; B.ln1b = wbuf[1]; B.wqkv = wbuf[2]; B.bqkv = wbuf[3]; B.wo = wbuf[4]; B.bo = wbuf[5];
  B.ln2g = wbuf[6]; B.ln2b = wbuf[7]; B.wup = wbuf[8]; B.bup = wbuf[9]; B.wdown = wbuf[10]; B.bdown = wbuf[11];
  CK(s.get(&B.kc, (size_t)H * S * d * D));
  CK(s.get(&B.vc, (size_t)H * S * d * D));
  CK(s.get(&B.n1, h * D));
  CK(s.get(&B.y, 3 * (size_t)h * D));
  CK(s.get(&B.q, h * D));
  CK(s.get(&B.lg, (size_t)H * S * D));
  CK(s.get(&B.ctx, h * D));
  CK(s.get(&B.attn, h * D));
  CK(s.get(&B.n2, h * D));
  CK(s.get(&B.act, mm * D));
  CK(s.get(&B.bad, sizeof(int)));
  CK(cudaMemset(B.bad, 0, sizeof(int)));
  return NFB_OK;
}

// history [H][len][d] (host) -> positions [0, len) of the [H][S][d] device cache
static int golden_load_cache(const GoldenBufs& B, const double* keys, const double* values, int H, int len, int S,
                             int d) {
  const size_t D = sizeof(double);
  for (int hh = 0; hh < H && len > 0; ++hh) {
    CK(cudaMemcpy(B.kc + (size_t)hh * S * d, keys + (size_t)hh * len * d, (size_t)len * d * D,
                  cudaMemcpyHostToDevice));
    CK(cudaMemcpy(B.vc + (size_t)hh * S * d, values + (size_t)hh * len * d, (size_t)len * d * D,
                  cudaMemcpyHostToDevice));
  }
  return NFB_OK;
}

static int golden_check_finite(const GoldenBufs& B) {
  int bad = 0;
  CK(cudaMemcpy(&bad, B.bad, sizeof(int), cudaMemcpyDeviceToHost));
  return bad ? fail(NFB_EINVAL, "non-finite activation") : NFB_OK;
}

// DecodeInstance.golden_logits (nf/fidelity.py:131-140): the float64 golden
// block (nf/golden.py:189-228) stepped over xs with a fresh cache from the
// prompt K/V, logits = unembed @ h per step (csrc/nfb_golden.cu).
int nfb_golden_logits(const nfb_model_desc* m, const nfb_block_weights* w, const double* unembed, const double* xs,
                      int steps, const double* prompt_k, const double* prompt_v, int prompt_len, double* logits) {
  if (!m || !w || !unembed || !xs || !logits || (prompt_len > 0 && (!prompt_k || !prompt_v)))
    return fail(NFB_EINVAL, "null argument");
  if (steps < 0 || prompt_len < 0) return fail(NFB_EINVAL, "steps and prompt_len must be >= 0");
  if (steps == 0) return NFB_OK;
  const int h = m->hidden, H = m->n_heads, d = m->d_head, V = m->vocab, S = prompt_len + steps;
  const size_t D = sizeof(double);
  DevScratch s;
  GoldenBufs B{};
  TRY(golden_setup(m, w, S, s, B));
  double *dx, *dout, *dun, *dlg;
  CK(s.get(&dx, (size_t)steps * h * D));
  CK(s.get(&dout, h * D));
  CK(s.get(&dun, (size_t)V * h * D));
  CK(s.get(&dlg, (size_t)steps * V * D));
  CK(cudaMemcpy(dx, xs, (size_t)steps * h * D, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dun, unembed, (size_t)V * h * D, cudaMemcpyHostToDevice));
  TRY(golden_load_cache(B, prompt_k, prompt_v, H, prompt_len, S, d));
  for (int t = 0; t < steps; ++t) {
    CK(golden_step(B, dx + (size_t)t * h, dout, h, H, d, m->d_mlp, m->rotary_dims, m->ln_eps, m->theta_base,
                   prompt_len + t, S, m->parallel_residual, m->gelu_exact, nullptr));
    CK(golden_probe(dun, dout, V, h, dlg + (size_t)t * V, nullptr));
  }
  TRY(golden_check_finite(B));
  CK(cudaMemcpy(logits, dlg, (size_t)steps * V * D, cudaMemcpyDeviceToHost));
  return NFB_OK;
}

// prefill_attention_tiled (nf/golden.py:234-265) for one head: Q, K, V
// [seq][d] float64 host arrays -> out [seq][d].
int nfb_prefill_attention_tiled(const double* Q, const double* K, const double* V, int seq, int d, int tile,
                                int causal, double scale, double* out) {
  if (!Q || !K || !V || !out) return fail(NFB_EINVAL, "null argument");
  if (seq < 0 || d < 1) return fail(NFB_EINVAL, "Q, K, V must share shape [seq, d_head]");
  if (tile < 1) return fail(NFB_EINVAL, "tile must be >= 1");
  if (seq == 0) return NFB_OK;
  const int t = tile < seq ? tile : seq;  // a tile wider than the sequence is the whole sequence
  if (((size_t)t + d) * sizeof(double) > 200 * 1024) return fail(NFB_EINVAL, "tile too large for shared memory");
  const size_t bytes = (size_t)seq * d * sizeof(double);
  DevScratch s;
  double *dq, *dk, *dv, *o;
  CK(s.get(&dq, bytes));
  CK(s.get(&dk, bytes));
  CK(s.get(&dv, bytes));
  CK(s.get(&o, bytes));
  CK(cudaMemcpy(dq, Q, bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk, K, bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, V, bytes, cudaMemcpyHostToDevice));
  CK(golden_prefill_tiled(dq, dk, dv, seq, d, t, causal ? 1 : 0, scale, o, nullptr));
  CK(cudaMemcpy(out, o, bytes, cudaMemcpyDeviceToHost));
  return NFB_OK;
}

// decoder_block_golden (nf/golden.py:189-228): one float64 golden step at
// pos = len over the history keys / values [H][len][d]; out [h], and the
// step's rotated K and V [H][d] for the caller's cache append.
int nfb_golden_block_step(const nfb_model_desc* m, const nfb_block_weights* w, const double* x, const double* keys,
                          const double* values, int len, double* out, double* k_new, double* v_new) {
  if (!m || !w || !x || !out || !k_new || !v_new || (len > 0 && (!keys || !values)))
    return fail(NFB_EINVAL, "null argument");
  if (len < 0) return fail(NFB_EINVAL, "len must be >= 0");
  const int h = m->hidden, H = m->n_heads, d = m->d_head, S = len + 1;
  const size_t D = sizeof(double);
  DevScratch s;
  GoldenBufs B{};
  TRY(golden_setup(m, w, S, s, B));
  double *dx, *dout;
  CK(s.get(&dx, h * D));
  CK(s.get(&dout, h * D));
  CK(cudaMemcpy(dx, x, h * D, cudaMemcpyHostToDevice));
  TRY(golden_load_cache(B, keys, values, H, len, S, d));
  CK(golden_step(B, dx, dout, h, H, d, m->d_mlp, m->rotary_dims, m->ln_eps, m->theta_base, len, S,
                 m->parallel_residual, m->gelu_exact, nullptr));
  TRY(golden_check_finite(B));
  CK(cudaMemcpy(out, dout, h * D, cudaMemcpyDeviceToHost));
  for (int hh = 0; hh < H; ++hh) {
    CK(cudaMemcpy(k_new + (size_t)hh * d, B.kc + ((size_t)hh * S + len) * d, d * D, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(v_new + (size_t)hh * d, B.vc + ((size_t)hh * S + len) * d, d * D, cudaMemcpyDeviceToHost));
  }
  return NFB_OK;
}

int nfb_output_project_atomic(const double* partials, const double* w_out, const double* b_out,
                              const double* residual, int n_blocks, int hidden, int fp16, uint64_t seed,
                              double* out) {
  if (!partials || !w_out || !b_out || !residual || !out) return fail(NFB_EINVAL, "null argument");
  if (n_blocks < 1 || hidden < 1) return fail(NFB_EINVAL, "n_blocks and hidden must be >= 1");
  const size_t h8 = (size_t)hidden * sizeof(double);
  DevScratch s;
  double *dp, *dw, *db, *dr, *pr, *o;
  int* ord;
  CK(s.get(&dp, n_blocks * h8));
  CK(s.get(&dw, hidden * h8));
  CK(s.get(&db, h8));
  CK(s.get(&dr, h8));
  CK(s.get(&pr, n_blocks * h8));
  CK(s.get(&ord, (size_t)hidden * n_blocks * sizeof(int)));
  CK(s.get(&o, h8));
  CK(cudaMemcpy(dp, partials, n_blocks * h8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw, w_out, hidden * h8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b_out, h8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dr, residual, h8, cudaMemcpyHostToDevice));
  CK(launch_project_atomic(dp, dw, db, dr, n_blocks, hidden, fp16 ? 1 : 0, seed, pr, ord, o, nullptr));
  CK(cudaMemcpy(out, o, h8, cudaMemcpyDeviceToHost));
  return NFB_OK;
}
}  // extern "C"
