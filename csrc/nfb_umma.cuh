// Shared host/device definitions of the batched-projection GEMM
// (csrc/nfb_umma.cu) and its consumers (csrc/nfb_batch.cu).
//
// Layouts (both "UMMA-native": K-major, SWIZZLE_128B canonical atoms of 8 rows
// x 128 bytes, 1024 B between atoms):
//   * blocked weights: W [M][K] -> blocks of 128 rows x 64 k (16 KB), block
//     (tile t, k-block kb) at byte (t * kb_count + kb) * 16384; inside a block
//     row r / 16-byte chunk c at r * 128 + ((c ^ (r & 7)) * 16).  A CTA's
//     stream-K range of (tile, k-block) units is therefore ONE contiguous byte
//     range: the producer streams it with 1-D bulk copies (no tensor maps, no
//     strided 128-byte rows).  Zero-padded to whole tiles / k-blocks.
//   * blocked activations: A [N][K] (N = n_pad rows, multiple of 8) -> per
//     k-block a [n_pad][64] block of n_pad * 128 bytes, same swizzle; written
//     directly in this layout by the kernels that produce them (LN, GELU, the
//     attention combine).
//   * output: the GEMM writes fp32 stream-K partials ws[tile][piece][n][128];
//     the consumer of Y sums the pieces of its tile in piece order (`uout`),
//     so the split-K fixup is deterministic and fully parallel and costs no
//     extra launch or in-kernel rendezvous.
#pragma once
#include <cstddef>
#include <cstdint>

namespace nfb {

constexpr int kUmmaM = 128;                      // weight rows per tile (UMMA M)
constexpr int kUmmaKB = 64;                      // k per block: one 128-byte swizzle row
constexpr int kUmmaBlk = kUmmaM * kUmmaKB * 2;   // bytes per weight block (16 KB)

// CTA owning global unit g under the stream-K split (start_i = floor(i*T/G)).
__host__ __device__ inline int u_owner(long long g, int G, int T) {
  return (int)(((g + 1) * (long long)G + T - 1) / T) - 1;
}

// Element index (fp16 units) of (row n, column k) in a blocked activation
// buffer with n_pad rows per k-block.
__host__ __device__ inline size_t ablk(int n, int k, int n_pad) {
  const int kb = k >> 6, c = (k >> 3) & 7, e = k & 7;
  return (size_t)kb * n_pad * 64 + (size_t)n * 64 + (size_t)(((c ^ (n & 7)) << 3) | e);
}

// Element index of (row m, column k) in a blocked weight buffer.
__host__ __device__ inline size_t wblk(int m, int k, int kbc) {
  const int t = m >> 7, r = m & 127, kb = k >> 6, c = (k >> 3) & 7, e = k & 7;
  return ((size_t)t * kbc + kb) * (kUmmaM * kUmmaKB) + (size_t)r * 64 + (size_t)(((c ^ (r & 7)) << 3) | e);
}

// Plan of one GEMM shape (host): Y[N][M] = W[M][K] . A[N][K]^T.
struct UPlan {
  int M, N, K;
  int n_pad;       // MMA N (multiple of 8, >= N)
  int kb;          // k-blocks per tile
  int tiles;       // m-tiles
  int total;       // tiles * kb stream-K units
  int G;           // CTAs
  int max_pieces;  // partial slots per tile
  int su;          // units (k-blocks) per ring stage
  int stages;      // ring stages
  size_t smem;     // dynamic shared memory
  size_t ws_floats() const { return (size_t)tiles * max_pieces * n_pad * kUmmaM; }
};

// Consumer view of a GEMM result (device): Y[n][m] = sum of the tile's pieces.
struct UOut {
  const float* ws;
  int n_pad, kb, total, G, max_pieces;
};

#ifdef __CUDACC__
__device__ __forceinline__ float uout(const UOut& o, int n, int m) {
  const int t = m >> 7, r = m & 127;
  const long long g0 = (long long)t * o.kb;
  const int first = u_owner(g0, o.G, o.total), last = u_owner(g0 + o.kb - 1, o.G, o.total);
  const float* p = o.ws + (((size_t)t * o.max_pieces) * o.n_pad + n) * kUmmaM + r;
  const size_t stride = (size_t)o.n_pad * kUmmaM;
  float acc = 0.f;
  for (int i = 0; i <= last - first; ++i) acc += __ldcg(p + i * stride);
  return acc;
}
// hi / lo activation rows b and B + b: y = W . (hi + lo)
__device__ __forceinline__ float uout2(const UOut& o, int b, int B, int m) {
  return uout(o, b, m) + uout(o, B + b, m);
}

// Programmatic dependent launch (PDL): wait for the predecessor grid's
// completion + memory, and let the successor grid be scheduled early.  Both
// are no-ops when the launch carried no programmatic-serialization attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

}  // namespace nfb
