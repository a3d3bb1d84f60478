// The reference's golden block (nf/golden.py:189-228) in float64 on the GPU,
// one decode step per call, for DecodeInstance.golden_logits
// (nf/fidelity.py:131-140).
//
// The golden pipeline is the unfused float64 restatement the fused kernel is
// judged against: weights used as given (no fp16 rounding), two-pass
// LayerNorm, f64 projections, partial RoPE with f64 angles, naive per-head
// softmax over the whole cache including the fresh token, tanh or erf GELU.
// Callers of the reference API (seed_sweep, fidelity studies) need it next to
// the kernel's logits; here it runs on the B200's native FP64 units instead
// of a CPU path.  Sizes are the fidelity instances' (hidden <= a few
// thousand), so the kernels are plain: one warp per output row for the
// matrix-vector products, one block per head for attention, one block for
// each LayerNorm.  Summation orders differ from numpy/BLAS, so results agree
// with the reference to float64 rounding (~1e-15 relative), not bitwise.
#include <cmath>
#include <cstdint>

#include <cuda_runtime.h>

#include "nfb_internal.h"

namespace nfb {

namespace {

__device__ __forceinline__ double warp_sum_g(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum_g(double v, double* sh) {
  v = warp_sum_g(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += sh[i];
  return t;
}

__device__ double block_max_g(double v, double* sh) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = -INFINITY;
  for (int i = 0; i < nw; ++i) t = fmax(t, sh[i]);
  return t;
}

// layernorm_two_pass (nf/golden.py:34-40): mean, then the population variance
// of the centered values; a non-finite input sets *bad (the reference raises
// ValueError("non-finite activation"), nf/golden.py:29-31).  One block.
__global__ void __launch_bounds__(256) ln_two_pass_kernel(const double* x, const double* g, const double* b, int n,
                                                          double eps, double* out, int* bad) {
  __shared__ double sh[32];
  double s = 0.0;
  int nf = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s += x[i];
    nf |= !isfinite(x[i]);
  }
  if (__syncthreads_or(nf) && threadIdx.x == 0) *bad = 1;
  const double mu = block_sum_g(s, sh) / n;
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += (x[i] - mu) * (x[i] - mu);
  const double var = block_sum_g(v, sh) / n;
  const double r = sqrt(var + eps);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = (x[i] - mu) / r * g[i] + b[i];
}

// y[r] = W[r] . x (+ bias[r]) (+ add[r]); act: 0 none, 1 GELU tanh, 2 GELU erf
// (nf/golden.py:156-166).  One warp per row.
__global__ void __launch_bounds__(256) gemv_kernel(const double* W, const double* x, const double* bias,
                                                   const double* add, int rows, int cols, int act, double* y) {
  const int lane = threadIdx.x & 31, r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const double* w = W + (size_t)r * cols;
  double s = 0.0;
  for (int k = lane; k < cols; k += 32) s += w[k] * x[k];
  s = warp_sum_g(s);
  if (lane) return;
  if (bias) s += bias[r];
  if (act == 1) s = 0.5 * s * (1.0 + tanh(0.79788456080286535588 * (s + 0.044715 * s * s * s)));
  if (act == 2) s = 0.5 * s * (1.0 + erf(s * 0.70710678118654752440));
  if (add) s += add[r];
  y[r] = s;
}

// q, k of every head rotated at `pos` (rope_partial, nf/golden.py:68-92:
// pairs (i, i + rd/2), angle pos * base^(-2i/rd), dims >= rd unchanged);
// k and v appended to the cache at `pos` (keys stored rotated,
// nf/weights.py:158-173).  y = [H][3d] interleaved QKV; grid H, block d.
__global__ void rope_append_kernel(const double* y, int H, int d, int rd, double base, int pos, int max_seq,
                                   double* q, double* kc, double* vc) {
  const int h = blockIdx.x, j = threadIdx.x, half = rd / 2;
  if (j >= d) return;
  const double* yh = y + (size_t)h * 3 * d;
  double qv = yh[j], kv = yh[d + j];
  if (j < rd) {
    const int i = j < half ? j : j - half;
    const double th = pos * pow(base, -2.0 * i / rd);
    const double c = cos(th), s = sin(th);
    if (j < half) {
      qv = yh[j] * c - yh[j + half] * s;
      kv = yh[d + j] * c - yh[d + j + half] * s;
    } else {
      qv = yh[j - half] * s + yh[j] * c;
      kv = yh[d + j - half] * s + yh[d + j] * c;
    }
  }
  q[(size_t)h * d + j] = qv;
  kc[((size_t)h * max_seq + pos) * d + j] = kv;
  vc[((size_t)h * max_seq + pos) * d + j] = yh[2 * d + j];
}

// attend_naive (nf/golden.py:139-150) per head over positions [0, P):
// logits = K q * scale, weights exp(logit - max), context = weights V / sum.
// Grid H, block 256; logits scratch [H][max_seq].
__global__ void __launch_bounds__(256) attend_kernel(const double* q, const double* kc, const double* vc, int d,
                                                     int P, int max_seq, double scale, double* lg,
                                                     double* ctx) {
  __shared__ double sh[32];
  const int h = blockIdx.x;
  const double* K = kc + (size_t)h * max_seq * d;
  const double* V = vc + (size_t)h * max_seq * d;
  const double* qh = q + (size_t)h * d;
  double* l = lg + (size_t)h * max_seq;
  double mx = -INFINITY;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += K[(size_t)p * d + j] * qh[j];
    s *= scale;
    l[p] = s;
    mx = fmax(mx, s);
  }
  const double m = block_max_g(mx, sh);
  double t = 0.0;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const double e = exp(l[p] - m);
    l[p] = e;
    t += e;
  }
  const double L = block_sum_g(t, sh);  // (barriers: every weight is visible below)
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double o = 0.0;
    for (int p = 0; p < P; ++p) o += l[p] * V[(size_t)p * d + j];
    ctx[(size_t)h * d + j] = o / L;
  }
}

// prefill_attention_tiled (nf/golden.py:234-265), one block per query row i:
// keys [0, limit) (limit = i + 1 causal, else seq) consumed in tiles of
// `tile` positions, each tile's two-pass softmax state (nf/golden.py:113-122)
// merged into the row's running state with the log-sum-exp rule
// (nf/golden.py:125-134; an empty running state takes the tile's as is).
// Dynamic shared memory: the tile's logits (tile doubles) + o [d].
__global__ void __launch_bounds__(128) prefill_tiled_kernel(const double* Q, const double* K, const double* V,
                                                            int seq, int d, int tile, int causal, double scale,
                                                            double* out) {
  extern __shared__ double psm[];
  __shared__ double sh[32];
  double* lg = psm;         // [tile]
  double* o = psm + tile;   // [d] running weighted values
  const int i = blockIdx.x, limit = causal ? i + 1 : seq;
  const double* q = Q + (size_t)i * d;
  double m = -INFINITY, l = 0.0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) o[j] = 0.0;
  for (int t0 = 0; t0 < limit; t0 += tile) {
    const int t1 = min(t0 + tile, limit);
    double mx = -INFINITY;
    for (int p = t0 + threadIdx.x; p < t1; p += blockDim.x) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += K[(size_t)p * d + j] * q[j];
      s *= scale;
      lg[p - t0] = s;
      mx = fmax(mx, s);
    }
    const double mt = block_max_g(mx, sh);
    double t = 0.0;
    for (int p = t0 + threadIdx.x; p < t1; p += blockDim.x) {
      const double e = exp(lg[p - t0] - mt);
      lg[p - t0] = e;
      t += e;
    }
    const double lt = block_sum_g(t, sh);  // (barriers: the weights are visible below)
    const double M = l == 0.0 ? mt : fmax(m, mt);
    const double fa = l == 0.0 ? 0.0 : exp(m - M), fb = l == 0.0 ? 1.0 : exp(mt - M);
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      double ot = 0.0;
      for (int p = t0; p < t1; ++p) ot += lg[p - t0] * V[(size_t)p * d + j];
      o[j] = l == 0.0 ? ot : o[j] * fa + ot * fb;
    }
    l = l == 0.0 ? lt : l * fa + lt * fb;
    m = M;
    __syncthreads();  // lg reused by the next tile
  }
  for (int j = threadIdx.x; j < d; j += blockDim.x) out[(size_t)i * d + j] = o[j] / l;
}

}  // namespace

cudaError_t golden_prefill_tiled(const double* Q, const double* K, const double* V, int seq, int d, int tile,
                                 int causal, double scale, double* out, cudaStream_t st) {
  const size_t smem = ((size_t)tile + d) * sizeof(double);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(prefill_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem);
    if (e != cudaSuccess) return e;
  }
  prefill_tiled_kernel<<<seq, 128, smem, st>>>(Q, K, V, seq, d, tile, causal, scale, out);
  return cudaGetLastError();
}

// One decoder_block_golden step (nf/golden.py:189-228) on device vectors:
// x [h] -> out [h]; the cache holds positions < pos and gains pos.
cudaError_t golden_step(const GoldenBufs& B, const double* x, double* out, int h, int H, int d, int m, int rd,
                        double eps, double base, int pos, int max_seq, int parallel, int gelu_exact,
                        cudaStream_t st) {
  const int wpb = 8;  // warps per 256-thread block (gemv)
  ln_two_pass_kernel<<<1, 256, 0, st>>>(x, B.ln1g, B.ln1b, h, eps, B.n1, B.bad);
  gemv_kernel<<<(3 * h + wpb - 1) / wpb, 256, 0, st>>>(B.wqkv, B.n1, B.bqkv, nullptr, 3 * h, h, 0, B.y);
  rope_append_kernel<<<H, (d + 31) / 32 * 32, 0, st>>>(B.y, H, d, rd, base, pos, max_seq, B.q, B.kc, B.vc);
  attend_kernel<<<H, 256, 0, st>>>(B.q, B.kc, B.vc, d, pos + 1, max_seq, 1.0 / sqrt((double)d), B.lg, B.ctx);
  // attn_res = x + W_out ctx + b_out
  gemv_kernel<<<(h + wpb - 1) / wpb, 256, 0, st>>>(B.wo, B.ctx, B.bo, x, h, h, 0, B.attn);
  ln_two_pass_kernel<<<1, 256, 0, st>>>(parallel ? x : B.attn, B.ln2g, B.ln2b, h, eps, B.n2, B.bad);
  gemv_kernel<<<(m + wpb - 1) / wpb, 256, 0, st>>>(B.wup, B.n2, B.bup, nullptr, m, h, gelu_exact ? 2 : 1, B.act);
  // out = attn_res + W_down act + b_down
  gemv_kernel<<<(h + wpb - 1) / wpb, 256, 0, st>>>(B.wdown, B.act, B.bdown, B.attn, h, m, 0, out);
  return cudaGetLastError();
}

// logits[r] = unembed[r] . hv (the probe head, nf/fidelity.py:139)
cudaError_t golden_probe(const double* unembed, const double* hv, int vocab, int h, double* logits, cudaStream_t st) {
  gemv_kernel<<<(vocab + 7) / 8, 256, 0, st>>>(unembed, hv, nullptr, nullptr, vocab, h, 0, logits);
  return cudaGetLastError();
}

}  // namespace nfb
