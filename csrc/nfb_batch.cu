// Batched decode (BASELINE.json configs[3]: Pythia-2.8B batch sweep 1/4/16/64,
// context 4096) -- B sequences at the same position, one token each per step.
//
// With B > 1 the projections become dense contractions: they run on our
// tcgen05 / TMEM GEMM (csrc/nfb_umma.cu) over blocked copies of the weights,
// fed with the activations split into fp16 hi + lo rows (x = hi + lo to
// ~2^-22, so the products keep fp32-class precision at the cost of a 2B-wide
// GEMM, still weight-bandwidth bound).  The kernels here write those rows
// directly in the GEMM's blocked SW128 layout (`ablk`) and read GEMM results
// through `uout`, which sums the stream-K pieces in fixed order (the split-K
// fixup, csrc/nfb_umma.cuh).  Every kernel opens with griddepcontrol.wait and
// (except the many-wave attention tiles) releases its successor at once, so
// under programmatic dependent launch the next GEMM's weight stream starts
// while the small kernels run.  Everything between the GEMMs
// (nf/golden.py:189-228 semantics):
//   ln_hilo_kernel        LN1 / LN2 (two-pass, nf/golden.py:34-40) -> hi/lo rows
//   attn_prep_kernel      QKV bias, partial RoPE (nf/golden.py:68-92), K/V append
//   attn_tile_kernel      decode attention over 128-position KV tiles (bulk-copied
//                         to shared memory), one softmax state per tile
//   attn_combine_kernel   log-sum-exp merge of the splits (nf/golden.py:128-136)
//   gelu_hilo_kernel      up bias + GELU (nf/golden.py:156-166) -> hi/lo rows
//   residual_kernel       x += W_o ctx + b_o + W_down g + b_down (parallel residual)
//   argmax_kernel         greedy token per sequence (nf/fidelity.py:27-34), vocab
//                         chunks + packed atomicMax; advance_kernel -> tokens
//   embed_kernel          token -> embedding row
#include <cuda_fp16.h>
#include <cstdint>

#include "nfb_internal.h"
#include "nfb_ptx.cuh"
#include "nfb_umma.cuh"

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

// Packed fp32x2 FMA (sm_100 FFMA2): a * b + c element-wise.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  const unsigned long long ab = (unsigned long long)__float_as_uint(a.x) | ((unsigned long long)__float_as_uint(a.y) << 32);
  const unsigned long long bb = (unsigned long long)__float_as_uint(b.x) | ((unsigned long long)__float_as_uint(b.y) << 32);
  const unsigned long long cb = (unsigned long long)__float_as_uint(c.x) | ((unsigned long long)__float_as_uint(c.y) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(ab), "l"(bb), "l"(cb));
  return make_float2(__uint_as_float((unsigned)d), __uint_as_float((unsigned)(d >> 32)));
}

// v -> blocked activation rows b (hi) and B + b (lo), column k
__device__ __forceinline__ void put_hilo(__half* a, int b, int B, int n_pad, int k, float v) {
  const __half hv = __float2half_rn(v);
  a[ablk(b, k, n_pad)] = hv;
  a[ablk(B + b, k, n_pad)] = __float2half_rn(v - __half2float(hv));
}

// grid B, block 256; x [B][h] fp32 (h <= 4096) -> A1 / A2 [2B][h] fp16 (rows
// b: hi, B + b: lo).  The row is read once into registers (4 float4 per
// thread), the LN parameters are fetched before the two reductions.
__device__ __forceinline__ float4 ld4(const float* p, int i4, bool ok) {
  return ok ? __ldg(reinterpret_cast<const float4*>(p) + i4) : make_float4(0.f, 0.f, 0.f, 0.f);
}
// columns 4 i4 .. 4 i4 + 3 (one half of a 16-byte chunk) of rows b / B + b
__device__ __forceinline__ void put_hilo4(__half* a, int b, int B, int n_pad, int i4, float4 v) {
  const __half2 h0 = __floats2half2_rn(v.x, v.y), h1 = __floats2half2_rn(v.z, v.w);
  const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
  __half2* hi = reinterpret_cast<__half2*>(a + ablk(b, 4 * i4, n_pad));
  __half2* lo = reinterpret_cast<__half2*>(a + ablk(B + b, 4 * i4, n_pad));
  hi[0] = h0;
  hi[1] = h1;
  lo[0] = __floats2half2_rn(v.x - f0.x, v.y - f0.y);
  lo[1] = __floats2half2_rn(v.z - f1.x, v.w - f1.y);
}
__global__ void __launch_bounds__(256) ln_hilo_kernel(const float* x, int B, int h, float eps, const float* g1,
                                                      const float* b1, const float* g2, const float* b2, __half* a1,
                                                      __half* a2, int n_pad) {
  __shared__ float sh[32];
  griddep_wait();
  griddep_launch();
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
    put_hilo4(a1, b, B, n_pad, i4,
              make_float4(n.x * G1[k].x + B1[k].x, n.y * G1[k].y + B1[k].y, n.z * G1[k].z + B1[k].z,
                          n.w * G1[k].w + B1[k].w));
    if (a2)
      put_hilo4(a2, b, B, n_pad, i4,
                make_float4(n.x * G2[k].x + B2[k].x, n.y * G2[k].y + B2[k].y, n.z * G2[k].z + B2[k].z,
                            n.w * G2[k].w + B2[k].w));
  }
}

// grid (B, H); y = the QKV GEMM (hi / lo rows) -> q [B][H][d] fp32 (rotated);
// rotated k and v appended at `pos` of kc / vc [B][H][max_seq][d].
__global__ void attn_prep_kernel(const UOut y, int B, int H, int d, int rd, const int* state, int max_seq,
                                 const float* bqkv, const float2* rope, float* q, __half* kc, __half* vc,
                                 int pos_step, size_t seq_stride) {
  griddep_wait();
  griddep_launch();
  // row b: position state[0] + b * pos_step (batch: 0, prefill: 1) of the
  // cache at kc + b * seq_stride (batch: own cache, prefill: the one cache)
  const int b = blockIdx.x, hh = blockIdx.y, h3 = 3 * H * d, pos = state[0] + b * pos_step;
  const float* bb = bqkv + (size_t)hh * 3 * d;
  extern __shared__ float sy[];  // [3d]
  (void)h3;
  for (int i = threadIdx.x; i < 3 * d; i += blockDim.x) sy[i] = uout2(y, b, B, hh * 3 * d + i) + bb[i];
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
#ifndef NFB_ATTN_TILE
#define NFB_ATTN_TILE 128
#endif
constexpr int kTile = NFB_ATTN_TILE;  // KV positions per attention block (128 measured best; 64: -4..-8 %)
// (tiles of 96 / 112 / 256 positions measured: +1 % / +0 % / -7..-14 %)
static_assert(kTile == 128, "attn_tile_kernel: one scoring thread per position of its kTile-thread block");
int attn_tile_positions() { return kTile; }
__global__ void __launch_bounds__(kTile) attn_tile_kernel(const float* q, const __half* kc, const __half* vc, int B,
                                                        int H, int d, int max_seq, const int* state,
                                                        float scale_log2, float* part, int pos_step,
                                                        size_t seq_stride) {
  griddep_wait();  // (no early release: this grid has many waves)
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
  // P.V partials of the groups [16][d] alias the K tile, dead after the
  // scores (the block reductions in between are barriers): 5 KB less shared
  // memory per block, so 5 instead of 4 blocks fit an SM
  float* so = reinterpret_cast<float*>(Ks);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sh + 32 + 2);
  const size_t base = (size_t)(bh / H) * seq_stride + ((size_t)(bh % H) * max_seq + p0) * d;
  // K and V on separate mbarriers: the scores start when K has landed
  // while V is still in flight
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
    const uint32_t bytes = (uint32_t)(n * d * 2);
    mbar_arrive_expect_tx(bar, bytes);
    mbar_arrive_expect_tx(bar + 1, bytes);
    const uint64_t pol = policy_evict_first();
    bulk_g2s(Ks, kc + base, bytes, bar, pol);
    bulk_g2s(Vs, vc + base, bytes, bar + 1, pol);
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
  mbar_wait(bar + 1, 0, nullptr, 30);
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
    float4* sv = reinterpret_cast<float4*>(so + grp * d + 8 * c8);  // two 16-byte stores (2-way, not 8-way, conflicts)
    sv[0] = make_float4(o8[0], o8[1], o8[2], o8[3]);
    sv[1] = make_float4(o8[4], o8[5], o8[6], o8[7]);
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

// Prefill variant (rows of one prompt chunk share the one cache, row r at
// position pos + r, causal): grid (H * ceil(T / kPrefillRows), S), block 128
// (4 warps).  The block bulk-copies its 128-position K / V tile ONCE for
// kPrefillRows consecutive rows (attn_tile_kernel re-fetched the same tile
// for every row of the chunk) and each warp scores whole rows on its own --
// lane L takes positions L, L + 32, L + 64, L + 96 (scores, warp-shuffle max /
// sum) and context elements L, L + 32, ... (P.V) -- so a row needs no block
// barrier.  Row r sees positions < pos + r + 1; its (m, l, o[d]) state goes
// to part in the layout attn_combine_kernel merges.
constexpr int kPrefillRows = 16;
__global__ void __launch_bounds__(kTile) attn_tile_rows_kernel(const float* q, const __half* kc, const __half* vc,
                                                             int T, int H, int d, int max_seq, const int* state,
                                                             float scale_log2, float* part) {
  griddep_wait();
  const int hh = blockIdx.x % H, r0 = (blockIdx.x / H) * kPrefillRows, s = blockIdx.y, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int r1 = min(T, r0 + kPrefillRows), pos = state[0], p0 = s * kTile;
  const int nmax = min(kTile, pos + r1 - p0);  // positions the last row sees in this tile
  if (nmax <= 0) {
    if (tid < r1 - r0) {
      float* out = part + ((size_t)((r0 + tid) * H + hh) * gridDim.y + s) * (d + 2);
      out[d] = -INFINITY;
      out[d + 1] = 0.f;
    }
    return;
  }
  extern __shared__ __align__(128) unsigned char tsm[];
  __half* Ks = reinterpret_cast<__half*>(tsm);
  __half* Vs = Ks + kTile * d;
  float* sq = reinterpret_cast<float*>(Vs + kTile * d);  // [4 warps][128]: the warp's q row (d <= 128)
  float* sp = sq + 4 * 128;                              // [4 warps][kTile] weights
  uint64_t* bar = reinterpret_cast<uint64_t*>(sp + 4 * kTile);
  const size_t base = ((size_t)hh * max_seq + p0) * d;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    const uint32_t bytes = (uint32_t)(nmax * d * 2);
    mbar_arrive_expect_tx(bar, 2 * bytes);
    const uint64_t pol = policy_evict_first();
    bulk_g2s(Ks, kc + base, bytes, bar, pol);
    bulk_g2s(Vs, vc + base, bytes, bar, pol);
  }
  __syncthreads();
  mbar_wait(bar, 0, nullptr, 31);
  const int cpr = d >> 3;
  float* wq = sq + warp * 128;
  float* wp = sp + warp * kTile;
  for (int r = r0 + warp; r < r1; r += 4) {
    const int n = min(kTile, pos + r + 1 - p0);
    float* out = part + ((size_t)(r * H + hh) * gridDim.y + s) * (d + 2);
    if (n <= 0) {
      if (lane == 0) {
        out[d] = -INFINITY;
        out[d + 1] = 0.f;
      }
      continue;
    }
    for (int i = lane; i < d; i += 32) wq[i] = q[((size_t)r * H + hh) * d + i];
    __syncwarp();
    float2 a[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    for (int c = 0; c < cpr; ++c) {
      const float4 q0 = *reinterpret_cast<const float4*>(wq + 8 * c);
      const float4 q1 = *reinterpret_cast<const float4*>(wq + 8 * c + 4);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint4 w = reinterpret_cast<const uint4*>(Ks + (size_t)(lane + 32 * k) * d)[c];
        const __half2* hp = reinterpret_cast<const __half2*>(&w);
        a[k] = ffma2(__half22float2(hp[0]), make_float2(q0.x, q0.y), a[k]);
        a[k] = ffma2(__half22float2(hp[1]), make_float2(q0.z, q0.w), a[k]);
        a[k] = ffma2(__half22float2(hp[2]), make_float2(q1.x, q1.y), a[k]);
        a[k] = ffma2(__half22float2(hp[3]), make_float2(q1.z, q1.w), a[k]);
      }
    }
    float sc[4], mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      sc[k] = lane + 32 * k < n ? (a[k].x + a[k].y) * scale_log2 : -INFINITY;
      mx = fmaxf(mx, sc[k]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float l = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float pw = lane + 32 * k < n ? exp2f(sc[k] - mx) : 0.f;
      wp[lane + 32 * k] = pw;
      l += pw;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    __syncwarp();
    // P.V: lane = (context chunk c8 of 8 elements, position group g); the
    // groups' partial sums are added in group order through shuffles
    const int ngrp = 32 / cpr, c8 = lane % cpr, g = lane / cpr;
    float2 o2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    if (g < ngrp) {
      const uint4* vr = reinterpret_cast<const uint4*>(Vs) + c8;
#pragma unroll 4
      for (int i = g; i < n; i += ngrp) {
        const uint4 w = vr[(size_t)i * cpr];
        const __half2* hp = reinterpret_cast<const __half2*>(&w);
        const float2 pw2 = make_float2(wp[i], wp[i]);
#pragma unroll
        for (int k = 0; k < 4; ++k) o2[k] = ffma2(pw2, __half22float2(hp[k]), o2[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 t = o2[k];
      for (int gg = 1; gg < ngrp; ++gg) {
        const float x = __shfl_sync(0xffffffffu, o2[k].x, min(31, lane + gg * cpr));
        const float y = __shfl_sync(0xffffffffu, o2[k].y, min(31, lane + gg * cpr));
        t.x += x;
        t.y += y;
      }
      o2[k] = t;
    }
    if (g == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        out[8 * c8 + 2 * k] = o2[k].x;
        out[8 * c8 + 2 * k + 1] = o2[k].y;
      }
    }
    if (lane == 0) {
      out[d] = mx;
      out[d + 1] = l;
    }
    __syncwarp();  // wq / wp reused by the warp's next row
  }
}

int attn_prefill_rows() { return kPrefillRows; }
size_t attn_tile_rows_smem(int d) { return (size_t)2 * kTile * d * 2 + (size_t)(4 * 128 + 4 * kTile) * 4 + 16; }

size_t attn_tile_smem(int d) { return (size_t)2 * kTile * d * 2 + (size_t)(d + kTile + 32 + 2) * 4 + 8 + 8; }

// grid B * H, block 128: merge the S split states in split order -> ctx
// [2B][h] fp16 hi / lo (blocked).  All states are read in one round (thread
// s < S fetches state s), then each context element sums its S terms.
__global__ void attn_combine_kernel(const float* part, int S, int B, int H, int d, __half* ctx, int n_pad) {
  __shared__ float sw[256], sh[32];
  griddep_wait();
  griddep_launch();
  const int bh = blockIdx.x, b = bh / H, hh = bh % H, tid = threadIdx.x;
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
    put_hilo(ctx, b, B, n_pad, hh * d + j, o / L);
  }
}

__device__ __forceinline__ float gelu_f(float x, int exact) {
  if (exact) return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
  const float k = 0.79788456080286536f;
  return 0.5f * x * (1.0f + tanhf(k * fmaf(0.044715f * x, x * x, x)));
}

// grid (B, ceil(m / 256)); u = the up GEMM (hi / lo rows) -> g hi / lo (blocked)
__global__ void gelu_hilo_kernel(const UOut u, int B, int m, const float* bup, int exact, __half* g, int n_pad) {
  griddep_wait();
  griddep_launch();
  const int b = blockIdx.x, i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const float v = uout2(u, b, B, i) + bup[i];
  put_hilo(g, b, B, n_pad, i, gelu_f(v, exact));
}

// grid (B, ceil(h / 256)); x += W_o ctx + b_o + W_down g + b_down (z, dn: GEMMs)
__global__ void residual_kernel(float* x, int B, int h, const UOut z, const float* bo, const UOut dn,
                                const float* bd) {
  griddep_wait();
  griddep_launch();
  const int b = blockIdx.x, i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= h) return;
  x[(size_t)b * h + i] += (uout2(z, b, B, i) + bo[i]) + (uout2(dn, b, B, i) + bd[i]);
}

// grid (B, chunks), block 256: logits (LM GEMM, hi / lo rows) -> per-block
// argmax over a vocab chunk -> packed 64-bit atomicMax of (ordered logit,
// ~index) into amax[b], so ties go to the lowest index like np.argmax
// (nf/fidelity.py:27-34).  advance_kernel turns amax into tokens.
__device__ __forceinline__ unsigned long long pack_argmax(float v, int idx) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)u << 32) | (unsigned long long)(0xffffffffu - (uint32_t)idx);
}
__global__ void __launch_bounds__(256) argmax_kernel(const UOut lg, int B, int V, unsigned long long* amax,
                                                     float* logits_out) {
  __shared__ unsigned long long sb[8];
  griddep_wait();
  griddep_launch();
  const int b = blockIdx.x, chunk = (V + gridDim.y - 1) / gridDim.y;
  const int i0 = blockIdx.y * chunk, i1 = min(V, i0 + chunk);
  unsigned long long best = 0ull;
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const float v = uout2(lg, b, B, i);
    if (logits_out) logits_out[(size_t)b * V + i] = v;
    const unsigned long long k = pack_argmax(v, i);
    best = k > best ? k : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  if ((threadIdx.x & 31) == 0) sb[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = sb[w] > best ? sb[w] : best;
    atomicMax(amax + b, best);
  }
}

// grid B: x[b] = embed[token[b]]
__global__ void embed_kernel(const int* tokens, const __half* embed, int h, int V, float* x) {
  griddep_wait();
  griddep_launch();
  const int b = blockIdx.x;
  int t = tokens[b];
  t = (t < 0 || t >= V) ? 0 : t;
  for (int i = threadIdx.x; i < h; i += blockDim.x) x[(size_t)b * h + i] = __half2float(embed[(size_t)t * h + i]);
}

// End of a step: position + 1; with the head, amax -> tokens (and amax
// cleared for the next step's atomicMax).
__global__ void advance_kernel(int* state, unsigned long long* amax, int* tokens, int B, int V) {
  griddep_wait();
  griddep_launch();
  for (int b = threadIdx.x; b < B && amax; b += blockDim.x) {
    const unsigned long long k = amax[b];
    int t = (int)(0xffffffffu - (uint32_t)(k & 0xffffffffull));
    tokens[b] = (t < 0 || t >= V) ? 0 : t;
    amax[b] = 0ull;
  }
  if (threadIdx.x == 0) state[0] += 1;
}

}  // namespace nfb
