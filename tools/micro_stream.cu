// Microbenchmark: HBM -> shared-memory stage ring exactly as the decode
// kernel streams it (148 CTAs in clusters of 2, 5 x 40 KB slots, 1-D bulk
// copies, one producer warp, 10 consumer warps), with a selectable amount of
// consumer work per stage.  Reports per-SM stage cadence and HBM GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I csrc -o tools/micro_stream tools/micro_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "nfb_ptx.cuh"

using namespace nfb;

constexpr int kSlots = 5, kSlotBytes = 40960, kNcw = 10;

__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

// MODE 0: wait/release only; 1: FFMA row-dots; 2: + butterfly shuffles;
// 3: tensor-core row-dot (16 m16n8k16 per warp per stage).  +10: no copies.
template <int MODE>
__global__ void __launch_bounds__(384, 1) stream(const uint4* src, size_t per_cta_bytes, int nstages, float* out,
                                                  long long* cyc, int* err) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSlots * kSlotBytes);
  uint64_t* empty = full + kSlots;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kNcw);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const unsigned char* base = reinterpret_cast<const unsigned char*>(src) + blockIdx.x * per_cta_bytes;
  const long long t0 = clock64();
  if (warp == kNcw) {
    uint64_t pol = policy_evict_first();
    int slot = 0;
    uint32_t ph = 0;
    for (int s = 0; s < nstages; ++s) {
      mbar_wait(&empty[slot], ph ^ 1u, err, 10);
      if (lane == 0) {
        if (MODE >= 10) {
          mbar_arrive(&full[slot]);
        } else {
          const size_t off = ((size_t)s * kSlotBytes) % per_cta_bytes;
          mbar_arrive_expect_tx(&full[slot], kSlotBytes);
          bulk_g2s(smem + slot * kSlotBytes, base + off, kSlotBytes, &full[slot], pol);
        }
      }
      __syncwarp();
      if (++slot == kSlots) {
        slot = 0;
        ph ^= 1u;
      }
    }
  } else if (warp < kNcw) {
    int slot = 0;
    uint32_t ph = 0;
    float acc = 0.f;
    const uint32_t ring = smem_u32(smem);
    float2 x2[4] = {{1.f, 0.5f}, {0.25f, 1.f}, {1.f, 2.f}, {0.5f, 0.5f}};
    for (int s = 0; s < nstages; ++s) {
      mbar_wait(&full[slot], ph, err, 20);
      constexpr int M = MODE % 10;
      if (M == 3) {
        const uint32_t b = ring + slot * kSlotBytes + warp * 4096 + lane * 16;
        float da[4] = {0.f, 0.f, 0.f, 0.f}, db[4] = {0.f, 0.f, 0.f, 0.f};
        uint4 w[8];
#pragma unroll
        for (int bi = 0; bi < 8; ++bi) w[bi] = lds128(b + bi * 512);
#pragma unroll
        for (int bi = 0; bi < 8; bi += 2) {
          mma_16816(da, lane, lane + 1, w[bi].x, w[bi].y);
          mma_16816(db, lane + 2, lane, w[bi + 1].x, w[bi + 1].y);
          mma_16816(da, lane, lane + 3, w[bi].z, w[bi].w);
          mma_16816(db, lane + 1, lane, w[bi + 1].z, w[bi + 1].w);
        }
        float t0 = da[0] + db[0];
        t0 += __shfl_down_sync(0xffffffffu, t0, 4);
        acc += t0;
      } else if (M >= 1) {
        const uint32_t b = ring + slot * kSlotBytes + tid * 16;
        float v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const uint4 w = lds128(b + r * 5120);
          const __half2* hp = reinterpret_cast<const __half2*>(&w);
          float a = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 t = __half22float2(hp[i]);
            a = fmaf(t.x, x2[i].x, a);
            a = fmaf(t.y, x2[i].y, a);
          }
          v[r] = a;
        }
        if (M >= 2) {
#pragma unroll
          for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[r] += __shfl_xor_sync(0xffffffffu, v[r], o);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) acc += v[r];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == kSlots) {
        slot = 0;
        ph ^= 1u;
      }
    }
    if (acc == 12345.f) out[0] = acc;
  }
  __syncthreads();
  if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
}

template <int MODE>
void run(const uint4* src, size_t per, int nst, float* out, long long* cyc, int* err, int smem, int cluster) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(stream<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, stream<MODE>, src, per, nst, out, cyc, err);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, stream<MODE>, src, per, nst, out, cyc, err);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double bytes = 148.0 * nst * kSlotBytes;
  printf("mode %d cluster %d: %.1f cycles/stage (CTA 0), %.3f ms, %.0f GB/s  [%s]\n", MODE, cluster,
         (double)h[0] / nst, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t per = 32ull << 20;  // 32 MB per CTA -> 4.7 GB total (>> L2)
  uint4* src;
  cudaMalloc(&src, per * 148);
  cudaMemset(src, 0, per * 148);
  float* out;
  long long* cyc;
  int* err;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&err, 4);
  const int nst = 4000;
  const int smem = kSlots * kSlotBytes + 256;
  for (int cl : {2}) {
    run<0>(src, per, nst, out, cyc, err, smem, cl);
    run<2>(src, per, nst, out, cyc, err, smem, cl);
    run<3>(src, per, nst, out, cyc, err, smem, cl);
    run<10>(src, per, nst, out, cyc, err, smem, cl);
    run<11>(src, per, nst, out, cyc, err, smem, cl);
    run<12>(src, per, nst, out, cyc, err, smem, cl);
    run<13>(src, per, nst, out, cyc, err, smem, cl);
  }
  return 0;
}
