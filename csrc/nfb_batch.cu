// Batched decode (BASELINE.json configs[3]: Pythia-2.8B batch sweep 1/4/16/64,
// context 4096) -- B sequences at the same position, one token each per step.
//
// With B > 1 the projections become dense contractions: they run as cuBLAS
// fp16 GEMMs (tensor cores, fp32 accumulation) over the weights in their
// decode-kernel layout, fed with the activations split into fp16 hi + lo rows
// (x = hi + lo to ~2^-22, so the products keep fp32-class precision at the
// cost of a 2B-wide GEMM, still weight-bandwidth bound).  Everything between
// the GEMMs is ours (nf/golden.py:189-228 semantics):
//   ln_hilo_kernel        LN1 / LN2 (two-pass, nf/golden.py:34-40) -> hi/lo rows
//   attn_prep_kernel      QKV bias, partial RoPE (nf/golden.py:68-92), K/V append
//   attn_split_kernel     split-KV decode attention, online softmax per split
//   attn_combine_kernel   log-sum-exp merge of the splits (nf/golden.py:128-136)
//   gelu_hilo_kernel      up bias + GELU (nf/golden.py:156-166) -> hi/lo rows
//   residual_kernel       x += W_o ctx + b_o + W_down g + b_down (parallel residual)
//   argmax_kernel         greedy token per sequence (nf/fidelity.py:27-34)
//   embed_kernel          token -> embedding row
#include <cuda_fp16.h>
#include <cstdint>

#include "nfb_internal.h"

namespace nfb {

__device__ __forceinline__ float block_sum(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += sh[i];
  return t;
}

__device__ __forceinline__ float block_max(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = -INFINITY;
  for (int i = 0; i < nw; ++i) t = fmaxf(t, sh[i]);
  return t;
}

__device__ __forceinline__ void put_hilo(__half* hi, __half* lo, int i, float v) {
  const __half a = __float2half_rn(v);
  hi[i] = a;
  lo[i] = __float2half_rn(v - __half2float(a));
}

// grid B; x [B][h] fp32 -> A1 / A2 [2B][h] fp16 (rows b: hi, B + b: lo)
__global__ void ln_hilo_kernel(const float* x, int B, int h, float eps, const float* g1, const float* b1,
                               const float* g2, const float* b2, __half* a1, __half* a2) {
  __shared__ float sh[32];
  const int b = blockIdx.x;
  const float* xb = x + (size_t)b * h;
  float s = 0.f;
  for (int i = threadIdx.x; i < h; i += blockDim.x) s += xb[i];
  const float mu = block_sum(s, sh) / h;
  float q = 0.f;
  for (int i = threadIdx.x; i < h; i += blockDim.x) q += (xb[i] - mu) * (xb[i] - mu);
  const float rstd = rsqrtf(block_sum(q, sh) / h + eps);
  for (int i = threadIdx.x; i < h; i += blockDim.x) {
    const float n = (xb[i] - mu) * rstd;
    put_hilo(a1 + (size_t)b * h, a1 + (size_t)(B + b) * h, i, n * g1[i] + b1[i]);
    if (a2) put_hilo(a2 + (size_t)b * h, a2 + (size_t)(B + b) * h, i, n * g2[i] + b2[i]);
  }
}

// grid (B, H); y [2B][3h] (hi / lo GEMM rows) -> q [B][H][d] fp32 (rotated);
// rotated k and v appended at `pos` of kc / vc [B][H][max_seq][d].
__global__ void attn_prep_kernel(const float* y, int B, int H, int d, int rd, const int* state, int max_seq,
                                 const float* bqkv, const float2* rope, float* q, __half* kc, __half* vc,
                                 int pos_step, size_t seq_stride) {
  // row b: position state[0] + b * pos_step (batch: 0, prefill: 1) of the
  // cache at kc + b * seq_stride (batch: own cache, prefill: the one cache)
  const int b = blockIdx.x, hh = blockIdx.y, h3 = 3 * H * d, pos = state[0] + b * pos_step;
  const float* yh = y + (size_t)b * h3 + (size_t)hh * 3 * d;
  const float* yl = y + (size_t)(B + b) * h3 + (size_t)hh * 3 * d;
  const float* bb = bqkv + (size_t)hh * 3 * d;
  extern __shared__ float sy[];  // [3d]
  for (int i = threadIdx.x; i < 3 * d; i += blockDim.x) sy[i] = yh[i] + yl[i] + bb[i];
  __syncthreads();
  const int half = rd >> 1;
  const float2* cs = rope + (size_t)pos * half;
  const size_t kvo = (size_t)b * seq_stride + ((size_t)hh * max_seq + pos) * d;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float qv = sy[j], kv = sy[d + j];
    if (j < rd) {
      const int i = j < half ? j : j - half;
      const float2 c = cs[i];
      if (j < half) {
        qv = sy[j] * c.x - sy[j + half] * c.y;
        kv = sy[d + j] * c.x - sy[d + j + half] * c.y;
      } else {
        qv = sy[j - half] * c.y + sy[j] * c.x;
        kv = sy[d + j - half] * c.y + sy[d + j] * c.x;
      }
    }
    q[((size_t)b * H + hh) * d + j] = qv;
    kc[kvo + j] = __float2half_rn(kv);
    vc[kvo + j] = __float2half_rn(sy[2 * d + j]);
  }
}

// grid (B * H, S), block 128: positions [s * per, min(P, (s+1) * per)) of
// sequence b / head hh; writes (m, l, o[d]) of the split to part.
__global__ void attn_split_kernel(const float* q, const __half* kc, const __half* vc, int B, int H, int d,
                                  int max_seq, const int* state, float scale_log2, float* part, int pos_step,
                                  size_t seq_stride) {
  // P = pos + 1 positions (history + the token appended by attn_prep_kernel;
  // prefill: causal, row b sees positions <= state[0] + b), split evenly
  // over gridDim.y blocks (nf/golden.py:234-265 for the prefill semantics)
  const int P = state[0] + (int)(blockIdx.x / H) * pos_step + 1, per = (P + gridDim.y - 1) / gridDim.y;
  extern __shared__ __align__(16) float sm[];
  float* sq = sm;           // [d]
  float* sp = sq + d;       // [128] scores / weights
  float* sh = sp + 128;     // [32] reduction scratch
  float* so = sh + 32;      // [16][d] P.V partials of the position groups
  const int bh = blockIdx.x, s = blockIdx.y;
  const int p0 = s * per, p1 = min(P, p0 + per);
  const __half* K = kc + (size_t)(bh / H) * seq_stride + (size_t)(bh % H) * max_seq * d;
  const __half* V = vc + (size_t)(bh / H) * seq_stride + (size_t)(bh % H) * max_seq * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) sq[i] = q[(size_t)bh * d + i];
  __syncthreads();
  // P.V: thread = (8-dim chunk c, position group g): 16-byte V loads
  const int cpr = d >> 3, ng = blockDim.x / cpr, c8 = threadIdx.x % cpr, grp = threadIdx.x / cpr;
  float m = -INFINITY, l = 0.f, o8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int t0 = p0; t0 < p1; t0 += 128) {
    const int pos = t0 + threadIdx.x;
    float sc = -INFINITY;
    if (pos < p1) {
      const uint4* kr = reinterpret_cast<const uint4*>(K + (size_t)pos * d);
      float a = 0.f;
      for (int c = 0; c < (d >> 3); ++c) {
        const uint4 w = __ldg(kr + c);
        const __half2* hp = reinterpret_cast<const __half2*>(&w);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __half22float2(hp[i]);
          a = fmaf(f.x, sq[8 * c + 2 * i], a);
          a = fmaf(f.y, sq[8 * c + 2 * i + 1], a);
        }
      }
      sc = a * scale_log2;
    }
    const float mn = fmaxf(m, block_max(sc, sh));
    const float pw = pos < p1 ? exp2f(sc - mn) : 0.f;
    sp[threadIdx.x] = pw;
    const float alpha = exp2f(m - mn);
    l = l * alpha + block_sum(pw, sh);  // (block_sum syncs: sp is visible below)
    m = mn;
    if (grp < ng) {
#pragma unroll
      for (int k = 0; k < 8; ++k) o8[k] *= alpha;
      const int n = min(128, p1 - t0);
      const uint4* vr = reinterpret_cast<const uint4*>(V + (size_t)t0 * d) + c8;
#pragma unroll 4
      for (int i = grp; i < n; i += ng) {
        const uint4 w = __ldg(vr + (size_t)i * cpr);
        const __half2* hp = reinterpret_cast<const __half2*>(&w);
        const float pw2 = sp[i];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __half22float2(hp[k]);
          o8[2 * k] = fmaf(pw2, f.x, o8[2 * k]);
          o8[2 * k + 1] = fmaf(pw2, f.y, o8[2 * k + 1]);
        }
      }
    }
    __syncthreads();
  }
  // combine the position groups (fixed order) -> o[d]
  if (grp < ng)
#pragma unroll
    for (int k = 0; k < 8; ++k) so[grp * d + 8 * c8 + k] = o8[k];
  __syncthreads();
  float* out = part + ((size_t)bh * gridDim.y + s) * (d + 2);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float t = 0.f;
    for (int g = 0; g < ng; ++g) t += so[g * d + j];
    out[j] = t;
  }
  if (threadIdx.x == 0) {
    out[d] = m;
    out[d + 1] = l;
  }
}

// grid B * H: merge S split states in split order -> ctx [2B][h] fp16 hi / lo
__global__ void attn_combine_kernel(const float* part, int S, int B, int H, int d, __half* ctx) {
  const int bh = blockIdx.x, b = bh / H, hh = bh % H, h = H * d;
  const float* pb = part + (size_t)bh * S * (d + 2);
  float M = -INFINITY;
  for (int s = 0; s < S; ++s)
    if (pb[s * (d + 2) + d + 1] > 0.f) M = fmaxf(M, pb[s * (d + 2) + d]);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    float L = 0.f, o = 0.f;
    for (int s = 0; s < S; ++s) {
      const float* st = pb + s * (d + 2);
      if (st[d + 1] > 0.f) {
        const float f = exp2f(st[d] - M);
        L += st[d + 1] * f;
        o += st[j] * f;
      }
    }
    put_hilo(ctx + (size_t)b * h, ctx + (size_t)(B + b) * h, hh * d + j, o / L);
  }
}

__device__ __forceinline__ float gelu_f(float x, int exact) {
  if (exact) return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
  const float k = 0.79788456080286536f;
  return 0.5f * x * (1.0f + tanhf(k * fmaf(0.044715f * x, x * x, x)));
}

// grid (B, ceil(m / 256)); u [2B][m] -> g [2B][m] fp16 hi / lo
__global__ void gelu_hilo_kernel(const float* u, int B, int m, const float* bup, int exact, __half* g) {
  const int b = blockIdx.x, i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const float v = u[(size_t)b * m + i] + u[(size_t)(B + b) * m + i] + bup[i];
  put_hilo(g + (size_t)b * m, g + (size_t)(B + b) * m, i, gelu_f(v, exact));
}

// grid (B, ceil(h / 256)); x += z_hi + z_lo + b_o + dn_hi + dn_lo + b_down
__global__ void residual_kernel(float* x, int B, int h, const float* z, const float* bo, const float* dn,
                                const float* bd) {
  const int b = blockIdx.x, i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= h) return;
  x[(size_t)b * h + i] += (z[(size_t)b * h + i] + z[(size_t)(B + b) * h + i] + bo[i]) +
                          (dn[(size_t)b * h + i] + dn[(size_t)(B + b) * h + i] + bd[i]);
}

// grid B: logits [2B][V] (hi / lo rows) -> argmax (lowest index on ties)
__global__ void argmax_kernel(const float* lg, int B, int V, int* tokens, float* logits_out) {
  __shared__ float sv[1024];
  __shared__ int si[1024];
  const int b = blockIdx.x;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = lg[(size_t)b * V + i] + lg[(size_t)(B + b) * V + i];
    if (logits_out) logits_out[(size_t)b * V + i] = v;
    if (v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x >> 1; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const float v = sv[threadIdx.x + s];
      const int j = si[threadIdx.x + s];
      if (v > sv[threadIdx.x] || (v == sv[threadIdx.x] && j < si[threadIdx.x])) {
        sv[threadIdx.x] = v;
        si[threadIdx.x] = j;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) tokens[b] = si[0];
}

// grid B: x[b] = embed[token[b]]
__global__ void embed_kernel(const int* tokens, const __half* embed, int h, int V, float* x) {
  const int b = blockIdx.x;
  int t = tokens[b];
  t = (t < 0 || t >= V) ? 0 : t;
  for (int i = threadIdx.x; i < h; i += blockDim.x) x[(size_t)b * h + i] = __half2float(embed[(size_t)t * h + i]);
}

__global__ void advance_pos_kernel(int* state) { state[0] += 1; }

}  // namespace nfb
