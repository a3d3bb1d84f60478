// Batched projections on the 5th-generation tensor cores (tcgen05 / TMEM / TMA).
//
// Y[n][m] = sum_k W[m][k] * A[n][k]  for the batched decode path (C4, B
// sequences) and prefill: W is a weight matrix in its reference row-major
// layout [M][K] (fp16, K-major), A the activation rows [N][K] (fp16 hi / lo
// rows, N = 2B), Y fp32.  Swap-AB: the weights are the UMMA M = 128 operand,
// the activations the N operand (N = 8 .. 256 in steps of 8), so a decode
// batch of any size is ONE instruction shape and the whole kernel streams the
// weight matrix once from HBM (the roofline: weights once + activations from
// L2).
//
// Per CTA (one per SM, persistent):
//   warp 0      TMA producer: W tile [128 rows x 64 k] and A tile [N x 64 k]
//               (cp.async.bulk.tensor.2d, SWIZZLE_128B, K-major) into a ring of
//               shared-memory stages, weights with an L2 evict-first hint;
//   warp 1      TMEM allocator + MMA issuer: one elected lane issues 4
//               tcgen05.mma.kind::f16 (K = 16 each) per stage into a TMEM
//               accumulator [128 lanes x N columns, fp32], tcgen05.commit frees
//               the stage; accumulators are double-buffered in TMEM so the next
//               piece's MMAs overlap the previous piece's epilogue;
//   warps 2..5  epilogue: tcgen05.ld (32x32b) TMEM -> registers -> global.
//
// Work split: "stream-K" over the (m-tile, k-block) space -- CTA i owns the
// contiguous k-block range [i*T/G, (i+1)*T/G) of the T = tiles * K/64 blocks,
// so every SM streams the same number of weight bytes whatever M is (W_out
// has 20 m-tiles for 148 SMs).  A tile covered by one CTA is written directly;
// a tile split between CTAs is fixed up deterministically: each piece stores
// its fp32 partial, the last piece to finish (atomic counter) sums the
// partials in piece order -- the result does not depend on arrival order, so
// the batched path stays bitwise reproducible run to run.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "nfb_internal.h"
#include "nfb_ptx.cuh"

namespace nfb {

constexpr int kUmmaM = 128;        // weight rows per tile (UMMA M)
constexpr int kUmmaKB = 64;        // k per stage: 64 fp16 = one 128-byte swizzle row
constexpr int kUmmaThreads = 192;  // 6 warps

struct UmmaArgs {
  int M, N, K;     // Y [N][M]
  int n_pad;       // MMA N (multiple of 8, >= N)
  int kb;          // k-blocks per tile
  int tiles;       // m-tiles
  int total;       // tiles * kb
  int stages;
  int max_pieces;  // partial slots per tile
  float* Y;
  float* ws;       // [tiles][max_pieces][n_pad][128] fp32 partials
  int* counters;   // [tiles], zero between launches
  int* err;
};

// ---- tcgen05 / TMA wrappers -----------------------------------------------
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
// 8 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Shared-memory matrix descriptor of a K-major SWIZZLE_128B tile (the layout
// TMA writes for a box of 64 fp16 x rows): 8-row x 128-byte swizzle atoms,
// SBO = 1024 B between atoms along M/N, LBO unused (1), version 1 (sm_100),
// layout type 2 (SWIZZLE_128B).  The start address advances by 32 B per
// K = 16 slice inside the 128-byte swizzle row.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor: D fp32, A/B fp16, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kUmmaM >> 4) << 24);
}

// CTA owning global k-block g under the stream-K split (start_i = floor(i*T/G)).
__device__ __forceinline__ int owner_cta(long long g, int G, int T) {
  return (int)(((g + 1) * G + T - 1) / T) - 1;
}

// Pieces of CTA `cta`: calls fn(tile, kk0, kk1, piece_index, piece_count).
template <class F>
__device__ __forceinline__ void for_each_piece(const UmmaArgs& a, int cta, int G, F&& fn) {
  const long long k0 = (long long)cta * a.total / G, k1 = (long long)(cta + 1) * a.total / G;
  for (long long g = k0; g < k1;) {
    const int tile = (int)(g / a.kb);
    const long long tend = (long long)(tile + 1) * a.kb;
    const long long e = k1 < tend ? k1 : tend;
    const int first = owner_cta((long long)tile * a.kb, G, a.total);
    const int last = owner_cta(tend - 1, G, a.total);
    fn(tile, (int)(g - (long long)tile * a.kb), (int)(e - (long long)tile * a.kb), cta - first, last - first + 1);
    g = e;
  }
}

__global__ void __launch_bounds__(kUmmaThreads, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap ta,
                     const UmmaArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment of the stage buffers (SWIZZLE_128B atoms)
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t wbytes = kUmmaM * kUmmaKB * 2, abytes = (uint32_t)a.n_pad * kUmmaKB * 2;
  const uint32_t stage_bytes = wbytes + abytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + (size_t)a.stages * stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + a.stages;
  uint64_t* tfull = bars + 2 * a.stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    tma_prefetch_desc(&tw);
    tma_prefetch_desc(&ta);
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  const int G = gridDim.x, cta = blockIdx.x;

  if (warp == 0) {
    // ---- TMA producer ----
    const uint64_t pol_w = policy_evict_first(), pol_a = policy_evict_last();
    int s = 0;
    uint32_t ph = 0;
    for_each_piece(a, cta, G, [&](int tile, int kk0, int kk1, int, int) {
      for (int kk = kk0; kk < kk1; ++kk) {
        if (lane == 0) {
          mbar_wait(&empty[s], ph ^ 1u, a.err, 40);
          const uint32_t fb = smem_u32(&full[s]);
          mbar_arrive_expect_tx_u32(fb, stage_bytes);
          const uint32_t dst = base + (uint32_t)s * stage_bytes;
          tma_load_2d(dst, &tw, kk * kUmmaKB, tile * kUmmaM, fb, pol_w);
          tma_load_2d(dst + wbytes, &ta, kk * kUmmaKB, 0, fb, pol_a);
        }
        __syncwarp();
        if (++s == a.stages) {
          s = 0;
          ph ^= 1u;
        }
      }
    });
  } else if (warp == 1) {
    // ---- MMA issuer ----
    const uint32_t idesc = idesc_f16(a.n_pad);
    int s = 0, p = 0;
    uint32_t ph = 0;
    for_each_piece(a, cta, G, [&](int, int kk0, int kk1, int, int) {
      const int buf = p & 1;
      const uint32_t d = tmem + (uint32_t)(buf * a.n_pad);
      // wait until the epilogue drained this accumulator buffer (piece p - 2)
      mbar_wait(&tempty[buf], (uint32_t)(((p >> 1) & 1) ^ 1), a.err, 41);
      tc_fence_after();
      for (int kk = kk0; kk < kk1; ++kk) {
        mbar_wait(&full[s], ph, a.err, 42);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = base + (uint32_t)s * stage_bytes;
#pragma unroll
          for (int k = 0; k < kUmmaKB / 16; ++k)
            umma_f16(d, sw128_desc(sa + 32u * k), sw128_desc(sa + wbytes + 32u * k), idesc,
                     (kk > kk0 || k > 0) ? 1u : 0u);
          umma_commit(smem_u32(&empty[s]));
          if (kk + 1 == kk1) umma_commit(smem_u32(&tfull[buf]));
        }
        __syncwarp();
        if (++s == a.stages) {
          s = 0;
          ph ^= 1u;
        }
      }
      ++p;
    });
  } else {
    // ---- epilogue (warps 2..5; warp w reads TMEM lanes 32 * (w % 4) ..) ----
    const int q = warp & 3;
    const int row = 32 * q + lane;  // row of the m-tile
    int p = 0;
    for_each_piece(a, cta, G, [&](int tile, int, int, int idx, int cnt) {
      const int buf = p & 1;
      mbar_wait(&tfull[buf], (uint32_t)((p >> 1) & 1), a.err, 43);
      tc_fence_after();
      const uint32_t t0 = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * a.n_pad);
      const int m = tile * kUmmaM + row;
      float* part = a.ws + ((size_t)tile * a.max_pieces + idx) * a.n_pad * kUmmaM;
      for (int c = 0; c < a.n_pad; c += 8) {
        float v[8];
        tmem_ld8(t0 + (uint32_t)c, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n = c + j;
          if (n >= a.N) break;
          if (cnt == 1) {
            if (m < a.M) a.Y[(size_t)n * a.M + m] = v[j];
          } else {
            __stcg(part + (size_t)n * kUmmaM + row, v[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      ++p;
      if (cnt > 1) {
        // deterministic split-tile fixup: the last piece to finish sums the
        // partials in piece order
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          __threadfence();
          const int old = atomicAdd(a.counters + tile, 1);
          *flag = old == cnt - 1;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (*reinterpret_cast<volatile int*>(flag)) {
          __threadfence();
          const float* tp = a.ws + (size_t)tile * a.max_pieces * a.n_pad * kUmmaM;
          if (m < a.M)
            for (int n = 0; n < a.N; ++n) {
              float acc = 0.f;
              for (int i = 0; i < cnt; ++i) acc += __ldcg(tp + ((size_t)i * a.n_pad + n) * kUmmaM + row);
              a.Y[(size_t)n * a.M + m] = acc;
            }
          if (threadIdx.x == 64) a.counters[tile] = 0;
        }
      }
    });
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, ncols);
  }
}

// ===========================================================================
// Host side
// ===========================================================================
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D fp16 K-major tensor map: `rows` rows of `k` elements (row stride
// `ld` elements), box [box_rows x 64], SWIZZLE_128B, zero fill out of bounds.
int make_tmap_f16(CUtensorMap* out, const void* base, uint64_t k, uint64_t rows, uint64_t ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return -1;
  const cuuint64_t dims[2] = {k, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kUmmaKB, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

bool umma_encoder_available() { return encode_fn() != nullptr; }

int umma_n_pad(int N) { return (N + 7) / 8 * 8; }

// Stream-K plan of one GEMM shape: grid and partial slots per tile.
void umma_plan(int M, int N, int K, int sm_count, int* grid, int* max_pieces) {
  const int tiles = (M + kUmmaM - 1) / kUmmaM, kb = (K + kUmmaKB - 1) / kUmmaKB;
  const long long T = (long long)tiles * kb;
  const int G = (int)(T < sm_count ? T : sm_count);
  int mp = 1;
  for (int t = 0; t < tiles; ++t) {
    auto owner = [&](long long g) { return (int)(((g + 1) * G + T - 1) / T) - 1; };
    const int c = owner((long long)(t + 1) * kb - 1) - owner((long long)t * kb) + 1;
    mp = c > mp ? c : mp;
  }
  *grid = G;
  *max_pieces = mp;
  (void)N;
}

size_t umma_smem(int n_pad, int* stages) {
  const size_t stage = (size_t)kUmmaM * kUmmaKB * 2 + (size_t)n_pad * kUmmaKB * 2;
  int s = (int)((200u * 1024u) / stage);
  if (s > 12) s = 12;
  if (s < 2) s = 2;
  *stages = s;
  return 1024 + s * stage + (2 * s + 4) * 8 + 16;
}

// Y[N][M] = W[M][K] . A[N][K]^T.  tw: tensor map of W (box 128 rows), ta: of A
// (box n_pad rows).  ws / counters: workspace of umma_plan's size.
cudaError_t umma_gemm(cudaStream_t st, const CUtensorMap* tw, const CUtensorMap* ta, int M, int N, int K, float* Y,
                      float* ws, int* counters, int* err, int sm_count) {
  UmmaArgs a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.n_pad = umma_n_pad(N);
  a.kb = (K + kUmmaKB - 1) / kUmmaKB;
  a.tiles = (M + kUmmaM - 1) / kUmmaM;
  a.total = a.tiles * a.kb;
  int grid = 0;
  umma_plan(M, N, K, sm_count, &grid, &a.max_pieces);
  const size_t smem = umma_smem(a.n_pad, &a.stages);
  a.Y = Y;
  a.ws = ws;
  a.counters = counters;
  a.err = err;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(umma_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  umma_gemm_kernel<<<grid, kUmmaThreads, smem, st>>>(*tw, *ta, a);
  return cudaGetLastError();
}

}  // namespace nfb

// ===========================================================================
// C-ABI diagnostics entry (include/nfb200.h): the batched-projection GEMM on
// caller-owned device buffers, for unit tests and microbenchmarks.
// ===========================================================================
namespace {
struct StandaloneWs {
  float* ws = nullptr;
  int* ctr = nullptr;
  int* err = nullptr;
  size_t ws_floats = 0;
  int ctr_n = 0;
};
StandaloneWs g_ws;  // grown on demand; the entry is not thread-safe
}  // namespace

extern "C" int nfb_gemm_f16_dev(int M, int N, int K, const void* W, const void* A, float* Y, void* stream) {
  using namespace nfb;
  if (M < 1 || N < 1 || N > 256 || K < 1 || K % 8 || !W || !A || !Y) return -1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = 0, mp = 0;
  umma_plan(M, N, K, sms, &grid, &mp);
  const int tiles = (M + kUmmaM - 1) / kUmmaM, np = umma_n_pad(N);
  const size_t need = (size_t)tiles * mp * np * kUmmaM;
  if (need > g_ws.ws_floats) {
    if (g_ws.ws) cudaFree(g_ws.ws);
    if (cudaMalloc(&g_ws.ws, need * 4) != cudaSuccess) return -2;
    g_ws.ws_floats = need;
  }
  if (tiles > g_ws.ctr_n) {
    if (g_ws.ctr) cudaFree(g_ws.ctr);
    if (cudaMalloc(&g_ws.ctr, (size_t)tiles * 4) != cudaSuccess) return -2;
    cudaMemset(g_ws.ctr, 0, (size_t)tiles * 4);
    g_ws.ctr_n = tiles;
  }
  if (!g_ws.err && (cudaMalloc(&g_ws.err, 4) != cudaSuccess || cudaMemset(g_ws.err, 0, 4) != cudaSuccess)) return -2;
  CUtensorMap tw, ta;
  if (make_tmap_f16(&tw, W, K, M, K, kUmmaM) || make_tmap_f16(&ta, A, K, N, K, np)) return -3;
  return umma_gemm((cudaStream_t)stream, &tw, &ta, M, N, K, Y, g_ws.ws, g_ws.ctr, g_ws.err, sms) == cudaSuccess ? 0 : -2;
}
