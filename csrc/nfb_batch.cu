// Batched decode (BASELINE.json configs[3]: Pythia-2.8B batch sweep 1/4/16/64,
// context 4096) -- B sequences at the same position, one token each per step.
//
// With B > 1 the projections become dense contractions: they run on our
// tcgen05 / TMEM / TMA GEMM (csrc/nfb_umma.cu) over the weights in their
// row-major layout, fed with the activations split into fp16 hi + lo rows
// (x = hi + lo to ~2^-22, so the products keep fp32-class precision at the
// cost of a 2B-wide GEMM, still weight-bandwidth bound).  Everything between
// the GEMMs is here too (nf/golden.py:189-228 semantics):
//   ln_hilo_kernel        LN1 / LN2 (two-pass, nf/golden.py:34-40) -> hi/lo rows
//   attn_prep_kernel      QKV bias, partial RoPE (nf/golden.py:68-92), K/V append
//   attn_tile_kernel      decode attention over 128-position KV tiles (bulk-copied
//                         to shared memory), one softmax state per tile
//   attn_combine_kernel   log-sum-exp merge of the splits (nf/golden.py:128-136)
//   gelu_hilo_kernel      up bias + GELU (nf/golden.py:156-166) -> hi/lo rows
//   residual_kernel       x += W_o ctx + b_o + W_down g + b_down (parallel residual)
//   argmax_kernel         greedy token per sequence (nf/fidelity.py:27-34)
//   embed_kernel          token -> embedding row
#include <cuda_fp16.h>
#include <cstdint>

#include "nfb_internal.h"
#include "nfb_ptx.cuh"

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

// grid B, block 256; x [B][h] fp32 (h <= 4096) -> A1 / A2 [2B][h] fp16 (rows
// b: hi, B + b: lo).  The row is read once into registers (4 float4 per
// thread), the LN parameters are fetched before the two reductions.
__device__ __forceinline__ float4 ld4(const float* p, int i4, bool ok) {
  return ok ? __ldg(reinterpret_cast<const float4*>(p) + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void put_hilo4(__half* hi, __half* lo, int i4, float4 v) {
  const __half2 h0 = __floats2half2_rn(v.x, v.y), h1 = __floats2half2_rn(v.z, v.w);
  const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
  reinterpret_cast<__half2*>(hi)[2 * i4] = h0;
  reinterpret_cast<__half2*>(hi)[2 * i4 + 1] = h1;
  reinterpret_cast<__half2*>(lo)[2 * i4] = __floats2half2_rn(v.x - f0.x, v.y - f0.y);
  reinterpret_cast<__half2*>(lo)[2 * i4 + 1] = __floats2half2_rn(v.z - f1.x, v.w - f1.y);
}
__global__ void __launch_bounds__(256) ln_hilo_kernel(const float* x, int B, int h, float eps, const float* g1,
                                                      const float* b1, const float* g2, const float* b2, __half* a1,
                                                      __half* a2) {
  __shared__ float sh[32];
  const int b = blockIdx.x, h4 = h >> 2;
  const float* xb = x + (size_t)b * h;
  float4 v[4], G1[4], B1[4], G2[4], B2[4];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i4 = threadIdx.x + k * blockDim.x;
    const bool ok = i4 < h4;
    v[k] = ok ? __ldcg(reinterpret_cast<const float4*>(xb) + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
    G1[k] = ld4(g1, i4, ok);
    B1[k] = ld4(b1, i4, ok);
    G2[k] = ld4(g2, i4, ok && a2);
    B2[k] = ld4(b2, i4, ok && a2);
    s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
  const float mu = block_sum(s, sh) / h;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (threadIdx.x + k * blockDim.x < h4) {
      const float dx = v[k].x - mu, dy = v[k].y - mu, dz = v[k].z - mu, dw = v[k].w - mu;
      q += (dx * dx + dy * dy) + (dz * dz + dw * dw);
    }
  const float rstd = rsqrtf(block_sum(q, sh) / h + eps);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i4 = threadIdx.x + k * blockDim.x;
    if (i4 >= h4) continue;
    const float4 n = make_float4((v[k].x - mu) * rstd, (v[k].y - mu) * rstd, (v[k].z - mu) * rstd,
                                 (v[k].w - mu) * rstd);
    put_hilo4(a1 + (size_t)b * h, a1 + (size_t)(B + b) * h, i4,
              make_float4(n.x * G1[k].x + B1[k].x, n.y * G1[k].y + B1[k].y, n.z * G1[k].z + B1[k].z,
                          n.w * G1[k].w + B1[k].w));
    if (a2)
      put_hilo4(a2 + (size_t)b * h, a2 + (size_t)(B + b) * h, i4,
                make_float4(n.x * G2[k].x + B2[k].x, n.y * G2[k].y + B2[k].y, n.z * G2[k].z + B2[k].z,
                            n.w * G2[k].w + B2[k].w));
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

// grid (B * H, S), block 128: one 128-position tile of sequence b / head hh.
// The tile's K and V rows (contiguous in the cache) arrive by two bulk copies
// (TMA engine, one mbarrier): the bytes in flight cost no registers, so every
// resident block has its whole tile outstanding.  Scores, max, exp2 weights
// and P.V from shared memory; writes the tile's (m, l, o[d]) to part.  Tiles
// at or past P (the grid covers max_seq) write an empty state.
constexpr int kTile = 128;
__global__ void __launch_bounds__(128) attn_tile_kernel(const float* q, const __half* kc, const __half* vc, int B,
                                                        int H, int d, int max_seq, const int* state,
                                                        float scale_log2, float* part, int pos_step,
                                                        size_t seq_stride) {
  const int bh = blockIdx.x, s = blockIdx.y, tid = threadIdx.x;
  const int P = state[0] + (bh / H) * pos_step + 1, p0 = s * kTile, n = min(kTile, P - p0);
  float* out = part + ((size_t)bh * gridDim.y + s) * (d + 2);
  if (n <= 0) {
    if (tid == 0) {
      out[d] = -INFINITY;
      out[d + 1] = 0.f;
    }
    return;
  }
  extern __shared__ __align__(128) unsigned char tsm[];
  __half* Ks = reinterpret_cast<__half*>(tsm);
  __half* Vs = Ks + kTile * d;
  float* sq = reinterpret_cast<float*>(Vs + kTile * d);  // [d]
  float* sp = sq + d;                                    // [128] weights
  float* sh = sp + kTile;                                // [32] reduction scratch
  float* so = sh + 32;                                   // [16][d] P.V partials of the groups
  uint64_t* bar = reinterpret_cast<uint64_t*>(so + 16 * d + 2);
  const size_t base = (size_t)(bh / H) * seq_stride + ((size_t)(bh % H) * max_seq + p0) * d;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    const uint32_t bytes = (uint32_t)(n * d * 2);
    mbar_arrive_expect_tx(bar, 2 * bytes);
    const uint64_t pol = policy_evict_first();
    bulk_g2s(Ks, kc + base, bytes, bar, pol);
    bulk_g2s(Vs, vc + base, bytes, bar, pol);
  }
  for (int i = tid; i < d; i += blockDim.x) sq[i] = q[(size_t)bh * d + i];
  __syncthreads();
  mbar_wait(bar, 0, nullptr, 30);  // watchdog: trap after 4 s like every other wait
  const int cpr = d >> 3;
  float sc = -INFINITY;
  if (tid < n) {
    const uint4* kr = reinterpret_cast<const uint4*>(Ks + (size_t)tid * d);
    float a = 0.f, a2 = 0.f;
    for (int c = 0; c < cpr; ++c) {
      const uint4 w = kr[c];
      const __half2* hp = reinterpret_cast<const __half2*>(&w);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(hp[i]);
        a = fmaf(f.x, sq[8 * c + 2 * i], a);
        a2 = fmaf(f.y, sq[8 * c + 2 * i + 1], a2);
      }
    }
    sc = (a + a2) * scale_log2;
  }
  const float m = block_max(sc, sh);
  const float pw = tid < n ? exp2f(sc - m) : 0.f;
  sp[tid] = pw;
  const float l = block_sum(pw, sh);  // (syncs: sp is visible below)
  const int ng = blockDim.x / cpr, c8 = tid % cpr, grp = tid / cpr;
  if (grp < ng) {
    float o8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const uint4* vr = reinterpret_cast<const uint4*>(Vs) + c8;
#pragma unroll 4
    for (int i = grp; i < n; i += ng) {
      const uint4 w = vr[(size_t)i * cpr];
      const __half2* hp = reinterpret_cast<const __half2*>(&w);
      const float pw2 = sp[i];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __half22float2(hp[k]);
        o8[2 * k] = fmaf(pw2, f.x, o8[2 * k]);
        o8[2 * k + 1] = fmaf(pw2, f.y, o8[2 * k + 1]);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) so[grp * d + 8 * c8 + k] = o8[k];
  }
  __syncthreads();
  for (int j = tid; j < d; j += blockDim.x) {
    float t = 0.f;
    for (int g = 0; g < ng; ++g) t += so[g * d + j];
    out[j] = t;
  }
  if (tid == 0) {
    out[d] = m;
    out[d + 1] = l;
  }
}

size_t attn_tile_smem(int d) { return (size_t)2 * kTile * d * 2 + (size_t)(d + kTile + 32 + 16 * d + 2) * 4 + 8; }

// grid B * H, block 128: merge the S split states in split order -> ctx
// [2B][h] fp16 hi / lo.  All states are read in one round (thread s < S
// fetches state s), then each context element sums its S terms.
__global__ void attn_combine_kernel(const float* part, int S, int B, int H, int d, __half* ctx) {
  __shared__ float sw[256], sh[32];
  const int bh = blockIdx.x, b = bh / H, hh = bh % H, h = H * d, tid = threadIdx.x;
  const float* pb = part + (size_t)bh * S * (d + 2);
  float ms = -INFINITY;
  for (int s = tid; s < S; s += blockDim.x) {
    const float l = pb[s * (d + 2) + d + 1];
    if (l > 0.f) {
      ms = fmaxf(ms, pb[s * (d + 2) + d]);
    }
  }
  const float M = block_max(ms, sh);
  float lsum = 0.f;
  for (int s = tid; s < S; s += blockDim.x) {
    const float l = pb[s * (d + 2) + d + 1];
    const float f = l > 0.f ? exp2f(pb[s * (d + 2) + d] - M) : 0.f;
    sw[s] = f;
    lsum += l > 0.f ? l * f : 0.f;
  }
  const float L = block_sum(lsum, sh);  // (syncs: sw is visible below)
  for (int j = tid; j < d; j += blockDim.x) {
    float o = 0.f;
#pragma unroll 8
    for (int s = 0; s < S; ++s) o += sw[s] == 0.f ? 0.f : pb[s * (d + 2) + j] * sw[s];
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

namespace nfb {

// out[c][r] = in[r][c] (fp16, rows x cols), 32 x 32 tiles
__global__ void transpose_f16_kernel(const __half* in, __half* out, int rows, int cols) {
  __shared__ __half tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[(size_t)r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[(size_t)c * rows + r] = tile[threadIdx.x][i];
  }
}

void transpose_f16(cudaStream_t st, const __half* in, __half* out, int rows, int cols) {
  transpose_f16_kernel<<<dim3((cols + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, st>>>(in, out, rows, cols);
}

}  // namespace nfb
