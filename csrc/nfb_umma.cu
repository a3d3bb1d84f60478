// Batched projections on the 5th-generation tensor cores (tcgen05 / TMEM).
//
// Y[n][m] = sum_k W[m][k] * A[n][k] for the batched decode path (C4, B
// sequences) and prefill: W a weight matrix, A the activation rows (fp16 hi /
// lo rows, N = 2B), fp32 result.  Swap-AB: the weights are the UMMA M = 128
// operand, the activations the N operand (8 .. 256 in steps of 8), so a
// decode batch of any size is ONE instruction shape and the kernel streams
// the weight matrix exactly once from HBM (the roofline: weights once +
// activations from L2).  Layouts and the output contract: csrc/nfb_umma.cuh.
//
// Per CTA (one per SM):
//   warp 0      producer (one lane): per unit (tile, k-block) one 16 KB 1-D
//               bulk copy of the blocked weight block -- a CTA's units are one
//               contiguous HBM range -- plus the unit's activation block
//               (L2-resident), into a ring of shared-memory stages, weights
//               with an L2 evict-first hint.  The first `stages` weight blocks
//               are issued BEFORE griddepcontrol.wait: under programmatic
//               dependent launch the weight stream starts while the previous
//               kernel of the chain (which produces A) is still running;
//   warp 1      TMEM allocator + MMA issuer: one lane issues 4 x
//               tcgen05.mma.kind::f16 (K = 16) per unit into a TMEM fp32
//               accumulator [128 lanes x n_pad columns]; tcgen05.commit frees
//               the stage; two accumulator buffers, so the next piece's MMAs
//               overlap the previous piece's epilogue;
//   warps 2..5  epilogue: tcgen05.ld (32x32b) TMEM -> registers -> the piece's
//               fp32 partial slot (coalesced 128-byte rows).
//
// Work split: stream-K over the tiles * k-blocks units (CTA i owns units
// [i*T/G, (i+1)*T/G)), so every SM streams the same number of weight bytes
// whatever M is (W_out has 20 m-tiles for 148 SMs).  The pieces of a split
// tile are summed by the consumer in piece order (`uout`): deterministic.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>

#include "nfb_internal.h"
#include "nfb_ptx.cuh"
#include "nfb_umma.cuh"

namespace nfb {

constexpr int kUmmaThreads = 192;  // 6 warps

struct UArgs {
  int N, n_pad, kb, total, stages, max_pieces;
  int su;                     // units (k-blocks) per stage
  uint32_t a_bytes;           // one activation block: n_pad * 128
  const unsigned char* Wb;    // blocked weights
  const unsigned char* Ab;    // blocked activations
  float* ws;                  // [tiles][max_pieces][n_pad][128]
  int* err;
  unsigned long long* trace;  // optional [G][8] globaltimer stamps (diagnostics)
};

// ---- tcgen05 wrappers -------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] . B[smem]^T, both K-major, fp16 in, fp32 accumulate.
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier when every previously issued tcgen05.mma of this
// thread has completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
// 8 consecutive fp32 columns of this thread's TMEM lane (no wait).
__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Shared-memory matrix descriptor of a K-major SWIZZLE_128B tile: 8-row x
// 128-byte swizzle atoms, SBO = 1024 B between atoms along M/N, LBO unused
// (1), version 1 (sm_100), layout type 2 (SWIZZLE_128B).  The start address
// advances by 32 B per K = 16 slice inside the 128-byte swizzle row.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor: D fp32, A/B fp16, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kUmmaM >> 4) << 24);
}

// Pieces of CTA `cta`: fn(tile, kk0, kk1, piece_index).
template <class F>
__device__ __forceinline__ void for_each_piece(const UArgs& a, int cta, int G, F&& fn) {
  const long long u0 = (long long)cta * a.total / G, u1 = (long long)(cta + 1) * a.total / G;
  for (long long g = u0; g < u1;) {
    const int tile = (int)(g / a.kb);
    const long long tend = (long long)(tile + 1) * a.kb;
    const long long e = u1 < tend ? u1 : tend;
    const int first = u_owner((long long)tile * a.kb, G, a.total);
    fn(tile, (int)(g - (long long)tile * a.kb), (int)(e - (long long)tile * a.kb), cta - first);
    g = e;
  }
}

__global__ void __launch_bounds__(kUmmaThreads, 1) umma_gemm_kernel(const UArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment of the stage buffers (SWIZZLE_128B atoms)
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t stage_bytes = (uint32_t)a.su * ((uint32_t)kUmmaBlk + a.a_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + (size_t)a.stages * stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + a.stages;
  uint64_t* tfull = bars + 2 * a.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  // the next kernel of the chain may be scheduled now (it waits for our
  // completion before touching anything we write)
  griddep_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * 8 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();
  const uint32_t ncols = a.n_pad * 2 <= 32 ? 32 : a.n_pad * 2 <= 64 ? 64 : a.n_pad * 2 <= 128 ? 128
                         : a.n_pad * 2 <= 256 ? 256 : 512;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  if (tr && threadIdx.x == 0) tr[1] = globaltimer();
  const int G = gridDim.x, cta = blockIdx.x;
  const long long u0 = (long long)cta * a.total / G, u1 = (long long)(cta + 1) * a.total / G;

  if (warp == 0) {
    // ---- producer: stage = up to `su` consecutive units, their weight blocks
    // in ONE bulk copy (a CTA's units are contiguous) and their activation
    // blocks in one copy per run of consecutive k-blocks (split only where a
    // tile boundary wraps kb back to 0).  Per SM the bulk engine completes
    // roughly one copy per ~0.3 us whatever its size (tools/micro_bulk.cu),
    // so bytes per copy, not copies in flight, set the streaming rate.
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first(), pol_a = policy_evict_last();
      const int su = a.su;
      const long long nst = (u1 - u0 + su - 1) / su;
      const int pre = (int)(nst < a.stages ? nst : a.stages);
      auto wcopy = [&](int st, long long u) {
        const int cnt = (int)(u1 - u < su ? u1 - u : su);
        const uint32_t fb = smem_u32(&full[st]);
        mbar_arrive_expect_tx_u32(fb, (uint32_t)cnt * ((uint32_t)kUmmaBlk + a.a_bytes));
        bulk_g2s_u32(base + (uint32_t)st * stage_bytes, a.Wb + (size_t)u * kUmmaBlk, (uint32_t)cnt * kUmmaBlk, fb,
                     pol_w);
      };
      auto acopy = [&](int st, long long u) {
        const int cnt = (int)(u1 - u < su ? u1 - u : su);
        const uint32_t fb = smem_u32(&full[st]), dst = base + (uint32_t)st * stage_bytes + (uint32_t)su * kUmmaBlk;
        for (int j = 0; j < cnt;) {
          const int kk = (int)((u + j) % a.kb);
          const int run = min(cnt - j, a.kb - kk);
          bulk_g2s_u32(dst + (uint32_t)j * a.a_bytes, a.Ab + (size_t)kk * a.a_bytes, (uint32_t)run * a.a_bytes, fb,
                       pol_a);
          j += run;
        }
      };
      // weights of the first `pre` stages: independent of the previous kernel
      for (int i = 0; i < pre; ++i) wcopy(i, u0 + (long long)i * su);
      if (tr) tr[2] = globaltimer();
      griddep_wait();  // A is written by the previous kernel
      for (int i = 0; i < pre; ++i) acopy(i, u0 + (long long)i * su);
      int st = pre == a.stages ? 0 : pre;
      uint32_t ph = pre == a.stages ? 1u : 0u;
      for (long long u = u0 + (long long)pre * su; u < u1; u += su) {
        mbar_wait(&empty[st], ph ^ 1u, a.err, 40);
        wcopy(st, u);
        acopy(st, u);
        if (++st == a.stages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- MMA issuer: per unit 4 x (M128 N n_pad K16); a new piece (tile)
    // switches the TMEM accumulator buffer, its last unit commits it to the
    // epilogue; the last unit of a stage commits the stage back to the producer.
    const uint32_t idesc = idesc_f16(a.n_pad);
    int st = 0, p = 0, j = 0, buf = 0;
    uint32_t ph = 0;
    for (long long u = u0; u < u1; ++u) {
      const int kk = (int)(u % a.kb);
      const bool piece_start = (u == u0) || kk == 0;
      const bool piece_end = (u + 1 == u1) || kk + 1 == a.kb;
      if (piece_start) {
        buf = p & 1;
        // wait until the epilogue drained this accumulator buffer (piece p - 2)
        mbar_wait(&tempty[buf], (uint32_t)(((p >> 1) & 1) ^ 1), a.err, 41);
        tc_fence_after();
      }
      if (j == 0) {
        mbar_wait(&full[st], ph, a.err, 42);
        if (tr && lane == 0 && u == u0) tr[3] = globaltimer();
        tc_fence_after();
      }
      if (lane == 0) {
        const uint32_t d = tmem + (uint32_t)(buf * a.n_pad);
        const uint32_t sw = base + (uint32_t)st * stage_bytes + (uint32_t)j * kUmmaBlk;
        const uint32_t sa = base + (uint32_t)st * stage_bytes + (uint32_t)a.su * kUmmaBlk + (uint32_t)j * a.a_bytes;
#pragma unroll
        for (int k = 0; k < kUmmaKB / 16; ++k)
          umma_f16(d, sw128_desc(sw + 32u * k), sw128_desc(sa + 32u * k), idesc, (!piece_start || k > 0) ? 1u : 0u);
        if (piece_end) umma_commit(smem_u32(&tfull[buf]));
        if (j + 1 == a.su || u + 1 == u1) umma_commit(smem_u32(&empty[st]));
      }
      __syncwarp();
      if (piece_end) ++p;
      if (++j == a.su || u + 1 == u1) {
        j = 0;
        if (++st == a.stages) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    if (tr && lane == 0) tr[4] = globaltimer();
  } else {
    // ---- epilogue (warps 2..5; warp w reads TMEM lanes 32 * (w % 4) ..) ----
    const int q = warp & 3;
    const int row = 32 * q + lane;  // row of the m-tile
    int p = 0;
    for_each_piece(a, cta, G, [&](int tile, int, int, int idx) {
      const int buf = p & 1;
      mbar_wait(&tfull[buf], (uint32_t)((p >> 1) & 1), a.err, 43);
      tc_fence_after();
      const uint32_t t0 = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * a.n_pad);
      float* part = a.ws + ((size_t)tile * a.max_pieces + idx) * a.n_pad * kUmmaM + row;
      for (int c = 0; c < a.n_pad; c += 32) {
        // up to 32 columns in flight, one wait
        uint32_t r[4][8];
        const int nc = (a.n_pad - c) >= 32 ? 4 : (a.n_pad - c) >> 3;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j < nc) tmem_ld8_nowait(t0 + (uint32_t)(c + 8 * j), r[j]);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int n = c + 8 * j + i;
            if (j < nc && n < a.N) __stcg(part + (size_t)n * kUmmaM, __uint_as_float(r[j][i]));
          }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      ++p;
    });
    if (tr && threadIdx.x == 64) tr[5] = globaltimer();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, ncols);
  }
  if (tr && threadIdx.x == 0) tr[6] = globaltimer();
}

// ---- layout conversion kernels -------------------------------------------
// Blocked copy of W: element (m, k) = trans ? src[k * ld + m] : src[m * ld + k]
// for m < M, k < K, zero elsewhere.  grid (tiles, kb), block 256: one 16 KB
// block, consecutive threads on consecutive rows (coalesced transposed reads).
__global__ void block_weights_kernel(const __half* src, int M, int K, size_t ld, int trans, __half* dst) {
  const int t = blockIdx.x, kb = blockIdx.y, kbc = gridDim.y;
  __half* out = dst + ((size_t)t * kbc + kb) * (kUmmaM * kUmmaKB);
  for (int i = threadIdx.x; i < kUmmaM * 8; i += blockDim.x) {
    const int r = i % kUmmaM, c = i / kUmmaM, m = t * kUmmaM + r, k0 = kb * kUmmaKB + c * 8;
    __align__(16) __half v[8];
    if (!trans && m < M && k0 + 8 <= K && (ld % 8) == 0) {
      *reinterpret_cast<uint4*>(v) = __ldg(reinterpret_cast<const uint4*>(src + (size_t)m * ld + k0));
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = k0 + e;
        v[e] = (m < M && k < K) ? (trans ? src[(size_t)k * ld + m] : src[(size_t)m * ld + k]) : __float2half(0.f);
      }
    }
    *reinterpret_cast<uint4*>(out + (size_t)r * 64 + ((c ^ (r & 7)) << 3)) = *reinterpret_cast<const uint4*>(v);
  }
}

// Blocked copy of row-major activations src [N][K] (n_pad rows, zero padded).
__global__ void block_act_kernel(const __half* src, int N, int n_pad, int K, int kbc, __half* dst) {
  const size_t total = (size_t)kbc * n_pad * 8;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int n = (int)(i % n_pad), c = (int)((i / n_pad) % 8), kb = (int)(i / ((size_t)n_pad * 8));
    __align__(16) __half v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = kb * kUmmaKB + c * 8 + e;
      v[e] = (n < N && k < K) ? src[(size_t)n * K + k] : __float2half(0.f);
    }
    *reinterpret_cast<uint4*>(dst + ablk(n, kb * kUmmaKB + c * 8, n_pad)) = *reinterpret_cast<const uint4*>(v);
  }
}

// Y[n][m] = uout(n, m) (diagnostics entry).
__global__ void uout_kernel(UOut o, int M, int N, float* Y) {
  const size_t total = (size_t)M * N;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / M), m = (int)(i % M);
    Y[i] = uout(o, n, m);
  }
}

// ===========================================================================
// Host side
// ===========================================================================
UPlan umma_plan(int M, int N, int K, int sm_count) {
  UPlan P{};
  P.M = M;
  P.N = N;
  P.K = K;
  P.n_pad = (N + 7) / 8 * 8;
  P.kb = (K + kUmmaKB - 1) / kUmmaKB;
  P.tiles = (M + kUmmaM - 1) / kUmmaM;
  P.total = P.tiles * P.kb;
  // 1.5 CTAs per SM: with the 80 KB ring two GEMM CTAs fit an SM, and the
  // extra CTAs fill SMs the other branch's kernels leave (C4 ctx 4096 B = 4 /
  // 16 / 64: +1.8 / +0.6 / +0.7 % over one per SM; 2 per SM and < 1 slower).
  int gmax = sm_count * 3 / 2;
  if (const char* e = getenv("NFB_UMMA_GRID")) gmax = atoi(e) > 0 ? std::min(atoi(e), sm_count * 2) : gmax;
  P.G = P.total < gmax ? P.total : gmax;
  int mp = 1;
  for (int t = 0; t < P.tiles; ++t) {
    const int c = u_owner((long long)(t + 1) * P.kb - 1, P.G, P.total) - u_owner((long long)t * P.kb, P.G, P.total) + 1;
    mp = c > mp ? c : mp;
  }
  P.max_pieces = mp;
  // units per stage
  // (measured: 16 KB single-unit stages beat 32 / 64 KB multi-unit stages in
  // the live batched step, B = 4: 3.15 vs 3.50 ms; NFB_UMMA_SU overrides)
  P.su = 1;
  if (const char* e = getenv("NFB_UMMA_SU")) P.su = atoi(e) < 1 ? 1 : (atoi(e) > 4 ? 4 : atoi(e));
  const size_t stage = (size_t)P.su * ((size_t)kUmmaBlk + (size_t)P.n_pad * kUmmaKB * 2);
  // Ring budget 80 KB, not the ~212 KB one CTA per SM could take: then the
  // attention tile blocks (47 KB) and the small kernels of the other branch
  // co-reside with the GEMM's CTAs, and the two branches of a layer really
  // overlap (C4 at ctx 4096, B = 4 / 16: 1298 -> 1571 / 2774 -> 3018 tok/s;
  // 64-96 KB equal, 40-48 KB and 128+ KB slower).  NFB_UMMA_SMEM_KB overrides.
  size_t budget = 80u * 1024u;
  if (const char* e = getenv("NFB_UMMA_SMEM_KB")) budget = (size_t)atoi(e) * 1024u;
  int s = (int)(budget / stage);
  if (s > 16) s = 16;
  if (s < 2) s = 2;
  P.stages = s;
  P.smem = 1024 + (size_t)s * stage + (2 * (size_t)s + 4) * 8 + 16;
  return P;
}

size_t umma_blocked_elems(int M, int K) {
  return (size_t)((M + kUmmaM - 1) / kUmmaM) * ((K + kUmmaKB - 1) / kUmmaKB) * kUmmaM * kUmmaKB;
}
size_t umma_act_elems(int n_pad, int K) { return (size_t)((K + kUmmaKB - 1) / kUmmaKB) * n_pad * kUmmaKB; }

UOut umma_out(const UPlan& P, const float* ws) { return UOut{ws, P.n_pad, P.kb, P.total, P.G, P.max_pieces}; }

void umma_block_weights(cudaStream_t st, const __half* src, int M, int K, size_t ld, bool trans, __half* dst) {
  block_weights_kernel<<<dim3((M + kUmmaM - 1) / kUmmaM, (K + kUmmaKB - 1) / kUmmaKB), 256, 0, st>>>(
      src, M, K, ld, trans ? 1 : 0, dst);
}

// Launch with the programmatic-serialization attribute (PDL) when `pdl`.
cudaError_t umma_gemm(cudaStream_t st, const UPlan& P, const void* Wb, const void* Ab, float* ws, int* err, bool pdl,
                      unsigned long long* trace) {
  UArgs a{};
  a.N = P.N;
  a.n_pad = P.n_pad;
  a.kb = P.kb;
  a.total = P.total;
  a.stages = P.stages;
  a.su = P.su;
  a.max_pieces = P.max_pieces;
  a.a_bytes = (uint32_t)P.n_pad * kUmmaKB * 2;
  a.Wb = static_cast<const unsigned char*>(Wb);
  a.Ab = static_cast<const unsigned char*>(Ab);
  a.ws = ws;
  a.err = err;
  a.trace = trace;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(umma_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.G, 1, 1);
  cfg.blockDim = dim3(kUmmaThreads, 1, 1);
  cfg.dynamicSmemBytes = P.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, umma_gemm_kernel, a);
}

}  // namespace nfb

// ===========================================================================
// C-ABI diagnostics entries (include/nfb200.h): the batched-projection GEMM on
// caller-owned device buffers, for unit tests and microbenchmarks.
// ===========================================================================
namespace {
struct StandaloneWs {
  float* ws = nullptr;
  __half* wb = nullptr;
  __half* ab = nullptr;
  int* err = nullptr;
  size_t ws_n = 0, wb_n = 0, ab_n = 0;
};
StandaloneWs g_ws;  // grown on demand; the entries are not thread-safe
unsigned long long* g_trace = nullptr;  // nfb_gemm_trace_dev: stamps of the next launches

template <class T>
bool grow(T** p, size_t* have, size_t need) {
  if (need <= *have) return true;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  if (cudaMalloc(reinterpret_cast<void**>(p), need * sizeof(T)) != cudaSuccess) return false;
  cudaMemset(*p, 0, need * sizeof(T));
  *have = need;
  return true;
}

int run_blocked(int M, int N, int K, const void* Wb, const void* A, float* Y, cudaStream_t st) {
  using namespace nfb;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const UPlan P = umma_plan(M, N, K, sms);
  if (!grow(&g_ws.ws, &g_ws.ws_n, P.ws_floats()) || !grow(&g_ws.ab, &g_ws.ab_n, umma_act_elems(P.n_pad, K)))
    return -2;
  if (!g_ws.err && (cudaMalloc(&g_ws.err, 4) != cudaSuccess || cudaMemset(g_ws.err, 0, 4) != cudaSuccess)) return -2;
  block_act_kernel<<<64, 256, 0, st>>>(static_cast<const __half*>(A), N, P.n_pad, K, P.kb, g_ws.ab);
  if (umma_gemm(st, P, Wb, g_ws.ab, g_ws.ws, g_ws.err, false, g_trace) != cudaSuccess) return -2;
  uout_kernel<<<296, 256, 0, st>>>(umma_out(P, g_ws.ws), M, N, Y);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
}  // namespace

extern "C" size_t nfb_gemm_blocked_bytes(int M, int K) {
  if (M < 1 || K < 1) return 0;
  return nfb::umma_blocked_elems(M, K) * 2;
}

extern "C" int nfb_gemm_block_weights_dev(int M, int K, const void* W, void* Wb, void* stream) {
  if (M < 1 || K < 1 || !W || !Wb) return -1;
  nfb::umma_block_weights((cudaStream_t)stream, static_cast<const __half*>(W), M, K, (size_t)K, false,
                          static_cast<__half*>(Wb));
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

extern "C" int nfb_gemm_f16_blocked_dev(int M, int N, int K, const void* Wb, const void* A, float* Y, void* stream) {
  if (M < 1 || N < 1 || N > 256 || K < 1 || !Wb || !A || !Y) return -1;
  return run_blocked(M, N, K, Wb, A, Y, (cudaStream_t)stream);
}

extern "C" int nfb_gemm_f16_dev(int M, int N, int K, const void* W, const void* A, float* Y, void* stream) {
  if (M < 1 || N < 1 || N > 256 || K < 1 || !W || !A || !Y) return -1;
  if (!grow(&g_ws.wb, &g_ws.wb_n, nfb::umma_blocked_elems(M, K))) return -2;
  const int r = nfb_gemm_block_weights_dev(M, K, W, g_ws.wb, stream);
  if (r) return r;
  return run_blocked(M, N, K, g_ws.wb, A, Y, (cudaStream_t)stream);
}

// Diagnostics: per-CTA globaltimer stamps [G][8] of the following standalone
// GEMM launches into a caller-owned device buffer (NULL: off).  Stamps: 0
// start, 1 setup done, 2 first weight copies issued, 3 first stage full
// (MMA warp), 4 last MMA issued, 5 epilogue done, 6 exit.
extern "C" int nfb_gemm_trace_dev(void* buf) {
  g_trace = static_cast<unsigned long long*>(buf);
  return 0;
}

// Host-only view of the GEMM plan (no device work): out[0..7] = grid, k-blocks
// per tile, tiles, max pieces per tile, ring stages, units per stage, n_pad,
// dynamic smem bytes.  For host-logic tests of the stream-K partition.
extern "C" int nfb_gemm_plan(int M, int N, int K, int sm_count, int* out) {
  if (M < 1 || N < 1 || N > 256 || K < 1 || sm_count < 1 || !out) return -1;
  const nfb::UPlan P = nfb::umma_plan(M, N, K, sm_count);
  out[0] = P.G;
  out[1] = P.kb;
  out[2] = P.tiles;
  out[3] = P.max_pieces;
  out[4] = P.stages;
  out[5] = P.su;
  out[6] = P.n_pad;
  out[7] = (int)P.smem;
  return 0;
}
