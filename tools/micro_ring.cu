// Microbenchmark: cost per stage of the producer -> consumer-warps mbarrier
// ring handshake (no data), as used by csrc/nfb_decode.cu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_ring tools/micro_ring.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ bool test_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ int g_flag;
template <int MODE>
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  if (MODE == 0) { while (!try_wait(b, ph)) {} }
  else if (MODE == 1) { while (!test_wait(b, ph)) {} }
  else if (MODE == 2) {  // the decode kernel's pattern: globaltimer watchdog
    if (try_wait(b, ph)) return;
    const unsigned long long t0 = gtimer();
    while (!try_wait(b, ph)) { if (gtimer() - t0 > 4000000000ull) g_flag = 1; }
  } else {  // clock64 watchdog
    if (try_wait(b, ph)) return;
    const long long t0 = clock64();
    while (!try_wait(b, ph)) { if (clock64() - t0 > 8000000000ll) g_flag = 1; }
  }
}

template <int MODE>
__global__ void ring(int nstages, int nslots, int ncw, long long* out) {
  __shared__ uint64_t full[16], empty[16];
  __shared__ int desc[16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], ncw); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp == ncw) {
    if (lane == 0) {
      int slot = 0; uint32_t ph = 0;
      for (int s = 0; s < nstages; ++s) {
        wait<MODE>(&empty[slot], ph ^ 1);
        desc[slot] = s;
        mbar_arrive(&full[slot]);
        if (++slot == nslots) { slot = 0; ph ^= 1; }
      }
    }
  } else if (warp < ncw) {
    int slot = 0; uint32_t ph = 0; int acc = 0;
    for (int s = 0; s < nstages; ++s) {
      wait<MODE>(&full[slot], ph);
      acc += desc[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == nslots) { slot = 0; ph ^= 1; }
    }
    if (acc == -1) out[1] = acc;
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  long long* d; cudaMalloc(&d, 148 * 8);
  long long h[148];
  const int N = 20000;
  const char* names[] = {"try_wait ", "test_wait", "try+gtimer", "try+clock64"};
  for (int mode = 0; mode < 4; ++mode)
    for (int ncw : {1, 4, 10}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) ring<0><<<148, (ncw + 1) * 32>>>(N, 5, ncw, d);
        else if (mode == 1) ring<1><<<148, (ncw + 1) * 32>>>(N, 5, ncw, d);
        else if (mode == 2) ring<2><<<148, (ncw + 1) * 32>>>(N, 5, ncw, d);
        else ring<3><<<148, (ncw + 1) * 32>>>(N, 5, ncw, d);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      printf("mode %s ncw %2d: %.1f cycles/stage\n", names[mode], ncw, (double)h[0] / N);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
