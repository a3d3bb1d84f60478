// Single-head split-KV attention and the atomic output projection of the
// reference's cluster simulator (nf/cluster.py:211-285), as device kernels.
//
// These are the reference's *unit-level* entry points of the fused block:
// `attend_split` (one head, KV history split over n_blocks contiguous ranges
// by the partition_kv rule, one partial softmax state per range, merged in the
// order the reduction strategy names) and `output_project_atomic` (per-block
// context shares projected through W_out and accumulated into residual +
// b_out, optionally modelling FP16 atomic adds: seed-keyed permuted order,
// binary16 rounding after every add).  The production decode kernel
// (nfb_decode.cu) does both inside its single launch per layer; these kernels
// expose the same algebra per call so code written against the reference's
// helpers runs on the GPU.  They compute in float64, the arithmetic the
// reference's helpers specify (B200 executes FP64 natively and the calls are
// tiny), so merge-order effects show at the same ulp level as in
// the reference.
//
// Layout: one CTA per KV range (split_state_kernel) writes its state
// {m, l, o[d]} to a [n_blocks][d + 2] scratch; merge_kernel has one thread per
// output column, each replaying the strategy's merge tree over its column
// (m and l are recomputed identically by every thread: no cross-thread
// communication, deterministic).  project_kernel: one warp per output
// element j.
#include <cuda_fp16.h>
#include <cstdint>
#include <math_constants.h>

namespace nfb {

namespace {

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// SplitMix64 output of the counter-th draw of the stream keyed by seed
// (nf/halfnum.py:35-45).
__device__ __forceinline__ uint64_t counter_rand(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Fisher-Yates permutation of range(n) keyed by seed (nf/halfnum.py:62-74).
__device__ void permutation(int n, uint64_t seed, int* idx) {
  for (int i = 0; i < n; ++i) idx[i] = i;
  uint64_t counter = 0;
  for (int i = n - 1; i > 0; --i) {
    const int j = (int)(counter_rand(seed, counter++) % (uint64_t)(i + 1));
    const int t = idx[i];
    idx[i] = idx[j];
    idx[j] = t;
  }
}

// Round through binary16 (RNE, one rounding from float64) and back: the
// reference's half_round_value (nf/halfnum.py:80-161).
__device__ __forceinline__ double half_round(double x) { return (double)__half2float(__double2half(x)); }

struct SState {
  double m, l, o;
};

// merge_states (nf/golden.py:128-136) on one output column.
__device__ __forceinline__ SState merge(SState a, SState b) {
  if (a.l == 0.0) return b;
  if (b.l == 0.0) return a;
  const double m = fmax(a.m, b.m);
  const double fa = exp(a.m - m), fb = exp(b.m - m);
  return {m, a.l * fa + b.l * fb, a.o * fa + b.o * fb};
}

// One CTA per KV range [a, e) of partition_kv(seq, n): the two-pass
// max-subtracted softmax state (nf/golden.py:116-125).  logits: [seq] scratch.
__global__ void __launch_bounds__(256) split_state_kernel(const double* __restrict__ q, const double* __restrict__ K,
                                                          const double* __restrict__ V, int seq, int d, int n,
                                                          double scale, double* __restrict__ logits,
                                                          double* __restrict__ states) {
  __shared__ double red[32];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int base = seq / n, extra = seq % n;
  const int a = b * base + min(b, extra), e = a + base + (b < extra ? 1 : 0);
  double* st = states + (size_t)b * (d + 2);
  if (a == e) {  // empty range (n_blocks > seq)
    for (int j = tid; j < d + 2; j += blockDim.x) st[j] = j == 0 ? -CUDART_INF : 0.0;
    return;
  }
  // logits = (K . q) * scale, one warp per key
  double mloc = -CUDART_INF;
  for (int i = a + warp; i < e; i += nw) {
    const double* k = K + (size_t)i * d;
    double s = 0.0;
    for (int j = lane; j < d; j += 32) s += k[j] * q[j];
    s = warp_sum_d(s) * scale;
    if (lane == 0) logits[i] = s;
    mloc = fmax(mloc, s);
  }
  if (lane == 0) red[warp] = mloc;
  __syncthreads();
  double m = red[0];
  for (int w = 1; w < nw; ++w) m = fmax(m, red[w]);
  __syncthreads();
  // weights and their sum
  double lsum = 0.0;
  for (int i = a + tid; i < e; i += blockDim.x) {
    const double w = exp(logits[i] - m);
    logits[i] = w;
    lsum += w;
  }
  lsum = warp_sum_d(lsum);
  if (lane == 0) red[warp] = lsum;
  __syncthreads();
  double l = 0.0;
  for (int w = 0; w < nw; ++w) l += red[w];
  // o = weights . V, one thread per column (coalesced across the row)
  for (int j = tid; j < d; j += blockDim.x) {
    double o = 0.0;
    for (int i = a; i < e; ++i) o += logits[i] * V[(size_t)i * d + j];
    st[2 + j] = o;
  }
  if (tid == 0) {
    st[0] = m;
    st[1] = l;
  }
}

// mode: 0 exact (closed form, nf/cluster.py:172-181), 1 ring, 2 tree, 3
// permuted (nf/cluster.py:184-201; order = permutation(n, seed)), 4 single
// block.  scratch: [d][n] SState per column thread (tree levels in place).
__global__ void __launch_bounds__(256) merge_kernel(const double* __restrict__ states, int n, int d, int mode,
                                                    uint64_t seed, int* __restrict__ order, SState* scratch,
                                                    double* __restrict__ out) {
  const int tid = threadIdx.x;
  if (mode == 3) {
    if (tid == 0) permutation(n, seed, order);
    __syncthreads();
  }
  for (int j = tid; j < d; j += blockDim.x) {
    auto S = [&](int i) {
      const double* s = states + (size_t)i * (d + 2);
      return SState{s[0], s[1], s[2 + j]};
    };
    SState r;
    if (mode == 4 || n == 1) {
      r = S(0);
    } else if (mode == 0) {
      double m = -CUDART_INF;
      bool any = false;
      for (int i = 0; i < n; ++i)
        if (S(i).l > 0.0) {
          m = fmax(m, S(i).m);
          any = true;
        }
      r = {any ? m : -CUDART_INF, 0.0, 0.0};
      for (int i = 0; i < n; ++i) {
        const SState s = S(i);
        if (s.l > 0.0) {
          const double f = exp(s.m - m);
          r.l += s.l * f;
          r.o += s.o * f;
        }
      }
    } else if (mode == 2) {
      SState* t = scratch + (size_t)j * n;
      for (int i = 0; i < n; ++i) t[i] = S(i);
      // level k holds its elements at indices 0, s, 2s, ... (s = 2^k): pair
      // (2t, 2t + 1) of the level is (2ts, (2t + 1)s); an odd last element
      // stays where it is -- the reference's level list, in place.
      for (int s = 1; s < n; s <<= 1)
        for (int i = 0; i + s < n; i += 2 * s) t[i] = merge(t[i], t[i + s]);
      r = t[0];
    } else {
      r = S(mode == 3 ? order[0] : 0);
      for (int k = 1; k < n; ++k) r = merge(r, S(mode == 3 ? order[k] : k));
    }
    out[j] = r.o / r.l;
  }
}

// Warp per output element j: projected[b] = partials[b] . W_out[j] (float64),
// then residual[j] + b_out[j] plus the contributions -- summed in block order
// (exact) or, fp16, added in the seed-keyed permuted order
// permutation(n, counter_rand(seed, j)) with binary16 rounding after every
// add (nf/cluster.py:253-285).  proj: [hidden][n], order: [hidden][n] scratch.
__global__ void __launch_bounds__(256) project_kernel(const double* __restrict__ P, const double* __restrict__ W,
                                                      const double* __restrict__ bias,
                                                      const double* __restrict__ residual, int n, int hidden,
                                                      int fp16, uint64_t seed, double* __restrict__ proj,
                                                      int* __restrict__ order, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= hidden) return;
  const double* w = W + (size_t)j * hidden;
  double* pj = proj + (size_t)j * n;
  for (int b = 0; b < n; ++b) {
    const double* p = P + (size_t)b * hidden;
    double s = 0.0;
    for (int k = lane; k < hidden; k += 32) s += p[k] * w[k];
    s = warp_sum_d(s);
    if (lane == 0) pj[b] = s;
  }
  if (lane) return;
  const double init = residual[j] + bias[j];
  if (!fp16 || n == 1) {
    double t = 0.0;
    for (int b = 0; b < n; ++b) t += pj[b];
    out[j] = init + t;
    return;
  }
  int* ord = order + (size_t)j * n;
  permutation(n, counter_rand(seed, (uint64_t)j), ord);
  double acc = half_round(init);
  for (int k = 0; k < n; ++k) acc = half_round(acc + pj[ord[k]]);
  out[j] = acc;
}

}  // namespace

cudaError_t launch_attend_split(const double* q, const double* K, const double* V, int seq, int d, int n, int mode,
                                uint64_t seed, double scale, double* logits, double* states, int* order,
                                void* scratch, double* out, cudaStream_t st) {
  split_state_kernel<<<n, 256, 0, st>>>(q, K, V, seq, d, n, scale, logits, states);
  merge_kernel<<<1, 256, 0, st>>>(states, n, d, mode, seed, order, static_cast<SState*>(scratch), out);
  return cudaGetLastError();
}

size_t attend_split_scratch_bytes(int n, int d) { return (size_t)n * d * sizeof(SState); }

cudaError_t launch_project_atomic(const double* P, const double* W, const double* bias, const double* residual,
                                  int n, int hidden, int fp16, uint64_t seed, double* proj, int* order, double* out,
                                  cudaStream_t st) {
  project_kernel<<<(hidden + 7) / 8, 256, 0, st>>>(P, W, bias, residual, n, hidden, fp16, seed, proj, order, out);
  return cudaGetLastError();
}

}  // namespace nfb
