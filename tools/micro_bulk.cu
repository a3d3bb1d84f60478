// Microbenchmark: per-SM throughput of 1-D bulk copies (cp.async.bulk, SASS
// UBLKCP) global -> shared memory, as a function of copy size, copies in
// flight and grid size, from HBM or from L2.  One producer lane issues into a
// ring of `slots` slots; one consumer warp waits on each slot's mbarrier and
// releases it (no compute).  Also: the same bytes with warp-wide LDG.128
// (MODE 1, 8 warps, 8 loads in flight per thread) for comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I csrc -o tools/micro_bulk tools/micro_bulk.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "nfb_ptx.cuh"

using namespace nfb;

__global__ void __launch_bounds__(64, 1) bulk_ring(const unsigned char* src, size_t per_cta, size_t wrap,
                                                   int copy_bytes, int slots, unsigned long long* t_out, int* err) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)slots * copy_bytes);
  uint64_t* empty = full + slots;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < slots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long n = (long long)(per_cta / copy_bytes);
  const size_t base = (size_t)blockIdx.x * per_cta;
  const unsigned long long t0 = globaltimer();
  if (tid == 0) {
    const uint64_t pol = policy_evict_first();
    int s = 0;
    uint32_t ph = 0;
    for (long long i = 0; i < n; ++i) {
      mbar_wait(&empty[s], ph ^ 1u, err, 1);
      mbar_arrive_expect_tx(&full[s], copy_bytes);
      bulk_g2s(smem + (size_t)s * copy_bytes, src + (base + (size_t)i * copy_bytes) % wrap, copy_bytes, &full[s], pol);
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
  } else if (tid == 32) {
    int s = 0;
    uint32_t ph = 0;
    for (long long i = 0; i < n; ++i) {
      mbar_wait(&full[s], ph, err, 2);
      mbar_arrive(&empty[s]);
      if (++s == slots) { s = 0; ph ^= 1u; }
    }
  }
  __syncthreads();
  if (tid == 0) {
    t_out[2 * blockIdx.x] = t0;
    t_out[2 * blockIdx.x + 1] = globaltimer();
  }
}

__global__ void __launch_bounds__(256, 1) ldg_stream(const uint4* src, size_t per_cta, size_t wrap, float* sink,
                                                     unsigned long long* t_out) {
  const size_t n16 = per_cta / 16, base = (size_t)blockIdx.x * (per_cta / 16), w16 = wrap / 16;
  const unsigned long long t0 = globaltimer();
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i < n16; i += 8 * blockDim.x) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const size_t j = i + (size_t)k * blockDim.x;
      v[k] = j < n16 ? __ldcs(src + (base + j) % w16) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  if (acc == 0x12345678u) sink[0] = 1.f;
  __syncthreads();
  if (threadIdx.x == 0) {
    t_out[2 * blockIdx.x] = t0;
    t_out[2 * blockIdx.x + 1] = globaltimer();
  }
}

int main() {
  const size_t big = (size_t)4 << 30;  // 4 GB source (HBM)
  unsigned char* src;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  unsigned long long* t;
  cudaMalloc(&t, 2 * 148 * 8);
  int* err;
  cudaMalloc(&err, 4);
  cudaMemset(err, 0, 4);
  float* sink;
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  unsigned long long h[2 * 148];
  auto report = [&](const char* what, int grid, size_t per_cta, int cb, int slots, const char* srcname) {
    cudaMemcpy(h, t, 2 * grid * 8, cudaMemcpyDeviceToHost);
    unsigned long long mn = ~0ull, mx = 0;
    double sum_rate = 0;
    for (int i = 0; i < grid; ++i) {
      mn = h[2 * i] < mn ? h[2 * i] : mn;
      mx = h[2 * i + 1] > mx ? h[2 * i + 1] : mx;
      sum_rate += per_cta / (double)(h[2 * i + 1] - h[2 * i]);
    }
    printf("{\"kind\":\"%s\",\"src\":\"%s\",\"grid\":%d,\"copy_kb\":%d,\"slots\":%d,\"inflight_kb\":%d,"
           "\"per_sm_GBps\":%.1f,\"total_GBps\":%.1f}\n",
           what, srcname, grid, cb / 1024, slots, cb * slots / 1024, sum_rate / grid, per_cta * (double)grid / (mx - mn));
  };
  const int grids[3] = {16, 74, 148};
  const int copies[4] = {4096, 16384, 40960, 65536};
  for (int src_l2 = 0; src_l2 < 2; ++src_l2) {
    const size_t wrap = src_l2 ? ((size_t)32 << 20) : big;  // 32 MB: L2-resident
    const char* sn = src_l2 ? "L2" : "HBM";
    for (int g : grids) {
      const size_t per_cta = src_l2 ? ((size_t)16 << 20) : (big / 148) / 65536 * 65536;
      for (int cb : copies)
        for (int inflight_kb : {32, 64, 128, 200}) {
          const int slots = inflight_kb * 1024 / cb;
          if (slots < 1 || slots > 64) continue;
          for (int rep = 0; rep < 2; ++rep)
            bulk_ring<<<g, 64, (size_t)slots * cb + 2 * slots * 8 + 64>>>(src, per_cta, wrap, cb, slots, t, err);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          report("bulk", g, per_cta, cb, slots, sn);
        }
      for (int rep = 0; rep < 2; ++rep) ldg_stream<<<g, 256>>>(reinterpret_cast<const uint4*>(src), per_cta, wrap, sink, t);
      cudaDeviceSynchronize();
      report("ldg", g, per_cta, 16, 8 * 256, sn);
    }
  }
  return 0;
}
