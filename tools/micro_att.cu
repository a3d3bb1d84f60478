// Microbenchmark of the tensor-core decode-attention stage (scores + online
// softmax + P.V over a 128-position K/V tile in shared memory), as used by
// csrc/nfb_decode.cu, on one CTA per SM with 10 consumer warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I csrc -o tools/micro_att tools/micro_att.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "nfb_ptx.cuh"

using namespace nfb;

constexpr int kNcw = 10, kD = 80, kN = 128;

__device__ __forceinline__ void mma_16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t h2_bits(__half2 v) { return *reinterpret_cast<uint32_t*>(&v); }
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t (&r)[2]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_trans(uint32_t addr, uint32_t (&r)[2]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t hilo(float a, float b, int g) {
  const __half2 hv = __floats2half2_rn(a, b);
  if (g == 0) return h2_bits(hv);
  if (g != 1) return 0u;
  const float2 hf = __half22float2(hv);
  return h2_bits(__floats2half2_rn(a - hf.x, b - hf.y));
}

template <int MODE>
__global__ void __launch_bounds__(384, 1) att(int nstages, float* out, long long* cyc) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nct = kNcw * 32;
  for (int i = tid; i < 2 * kN * kD; i += blockDim.x)
    reinterpret_cast<__half*>(smem)[i] = __float2half(0.01f * ((i * 37) % 101 - 50));
  float* scb = reinterpret_cast<float*>(smem + 2 * kN * kD * 2);
  __syncthreads();
  if (warp >= kNcw) return;
  const int g = lane >> 2, c = lane & 3;
  uint32_t qa[5][2];
  for (int st = 0; st < 5; ++st) {
    qa[st][0] = hilo(0.1f * lane, 0.2f, g);
    qa[st][1] = hilo(0.3f, 0.01f * st, g);
  }
  float dv[4] = {0.f, 0.f, 0.f, 0.f}, am = -INFINITY, al = 0.f;
  const uint32_t sb = smem_u32(smem);
  const long long t0 = clock64();
  long long tsc = 0, tmax = 0, tpv = 0;
  for (int it = 0; it < nstages; ++it) {
    const int n = kN, apos0 = it * 7;
    const int d = kD, nc = d >> 3, KS = d >> 4;
    const uint32_t rowb = d * 2, Kb = sb, Vb = sb + n * rowb;
    float* sc = scb + (it & 1) * kN;
    const long long c0 = clock64();
    long long c1, c2;
    if (MODE >= 6) {
      __half* phi = reinterpret_cast<__half*>(scb + 2 * kN);
      __half* plo = phi + kN;
      const int nb8 = (n + 7) >> 3;
      for (int blk = warp; blk < nb8; blk += 2 * kNcw) {
        const int blk2 = blk + kNcw;
        const bool two = blk2 < nb8;
        float D[4] = {0.f, 0.f, 0.f, 0.f}, E[4] = {0.f, 0.f, 0.f, 0.f};
        const int r8 = lane & 7, mi = lane >> 3;
        const int prow = blk * 8 + r8, prow2 = blk2 * 8 + r8;
        const uint32_t ra = Kb + prow * rowb, ra2 = Kb + prow2 * rowb;
        const int rot = (apos0 + prow) % nc, rot2 = (apos0 + prow2) % nc;
#pragma unroll
        for (int st = 0; st < 5; st += 2) {
          const int ch = 2 * st + (st + 1 < KS ? mi : (mi & 1));
          int c1_ = ch + rot; c1_ = c1_ >= nc ? c1_ - nc : c1_;
          int c2_ = ch + rot2; c2_ = c2_ >= nc ? c2_ - nc : c2_;
          if (st + 1 < KS) {
            uint32_t b[4], e[4];
            ldsm_x4(ra + c1_ * 16, b);
            if (two) ldsm_x4(ra2 + c2_ * 16, e);
            mma_16816(D, qa[st][0], qa[st][1], b[0], b[1]);
            if (two) mma_16816(E, qa[st][0], qa[st][1], e[0], e[1]);
            mma_16816(D, qa[st + 1][0], qa[st + 1][1], b[2], b[3]);
            if (two) mma_16816(E, qa[st + 1][0], qa[st + 1][1], e[2], e[3]);
          } else {
            uint32_t b[2], e[2];
            ldsm_x2(ra + c1_ * 16, b);
            if (two) ldsm_x2(ra2 + c2_ * 16, e);
            mma_16816(D, qa[st][0], qa[st][1], b[0], b[1]);
            if (two) mma_16816(E, qa[st][0], qa[st][1], e[0], e[1]);
          }
        }
        const float t0_ = D[0] + __shfl_down_sync(0xffffffffu, D[0], 4);
        const float t1_ = D[1] + __shfl_down_sync(0xffffffffu, D[1], 4);
        const float u0_ = E[0] + __shfl_down_sync(0xffffffffu, E[0], 4);
        const float u1_ = E[1] + __shfl_down_sync(0xffffffffu, E[1], 4);
        if (lane < 4) {
          const int pp = blk * 8 + 2 * lane;
          sc[pp] = pp < n ? t0_ * 0.16f : -INFINITY;
          sc[pp + 1] = pp + 1 < n ? t1_ * 0.16f : -INFINITY;
          if (two) {
            const int qq = blk2 * 8 + 2 * lane;
            sc[qq] = qq < n ? u0_ * 0.16f : -INFINITY;
            sc[qq + 1] = qq + 1 < n ? u1_ * 0.16f : -INFINITY;
          }
        }
      }
      c1 = clock64();
      consumer_sync(nct);
      float mx = -INFINITY;
      for (int i = lane; i < n; i += 32) mx = fmaxf(mx, sc[i]);
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
      const float mn = fmaxf(am, mx);
      const float alpha = fast_exp2(am - mn);
      const int nk = (n + 15) >> 4;
      for (int t = tid; t < 16 * nk; t += nct) {
        const float pv = t < n ? fast_exp2(sc[t] - mn) : 0.f;
        const __half hv = __float2half_rn(pv);
        phi[t] = hv;
        plo[t] = __float2half_rn(pv - __half2float(hv));
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) dv[k] *= alpha;
      consumer_sync(nct);
      c2 = clock64();
      const int g = lane >> 2, c = lane & 3;
      const __half* src = g == 0 ? phi : plo;
      float lsum = 0.f;
      float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (MODE == 6 && j >= nk) break;
        if (j >= nk) continue;
        const int q0 = 16 * j + 2 * c;
        const uint32_t a0 = g < 2 ? *reinterpret_cast<const uint32_t*>(src + q0) : 0u;
        const uint32_t a2 = g < 2 ? *reinterpret_cast<const uint32_t*>(src + q0 + 8) : 0u;
        const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&a0));
        const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(&a2));
        lsum += (f0.x + f0.y) + (f2.x + f2.y);
        const int prow = 16 * j + (lane & 15);
        int ch = warp + (apos0 + prow) % nc;
        ch = ch >= nc ? ch - nc : ch;
        uint32_t b[2];
        ldsm_x2_trans(Vb + prow * rowb + ch * 16, b);
        const uint32_t m0 = (q0 < n ? 0xffffu : 0u) | (q0 + 1 < n ? 0xffff0000u : 0u);
        const uint32_t m1 = (q0 + 8 < n ? 0xffffu : 0u) | (q0 + 9 < n ? 0xffff0000u : 0u);
        if (j & 1) mma_16816(e, a0, a2, b[0] & m0, b[1] & m1);
        else mma_16816(dv, a0, a2, b[0] & m0, b[1] & m1);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) dv[k] += e[k];
#pragma unroll
      for (int o2 = 1; o2 < 8; o2 <<= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o2);
      al = al * alpha + __shfl_sync(0xffffffffu, lsum, 0);
      am = mn;
    } else {
    const int nb8 = (n + 7) >> 3;
    for (int blk = warp; blk < nb8; blk += kNcw) {
      float D[4] = {0.f, 0.f, 0.f, 0.f};
      const int prow = blk * 8 + (lane & 7), mi = lane >> 3;
      const uint32_t ra = Kb + prow * rowb;
      const int rot = (apos0 + prow) % nc;
#pragma unroll
      for (int st = 0; st < 5; st += 2) {
        if (st + 1 < KS) {
          uint32_t b[4];
          ldsm_x4(ra + (((2 * st + mi + rot) % nc) * 16), b);
          mma_16816(D, qa[st][0], qa[st][1], b[0], b[1]);
          mma_16816(D, qa[st + 1][0], qa[st + 1][1], b[2], b[3]);
        } else {
          uint32_t b[2];
          ldsm_x2(ra + (((2 * st + (mi & 1) + rot) % nc) * 16), b);
          mma_16816(D, qa[st][0], qa[st][1], b[0], b[1]);
        }
      }
      const float t0_ = D[0] + __shfl_down_sync(0xffffffffu, D[0], 4);
      const float t1_ = D[1] + __shfl_down_sync(0xffffffffu, D[1], 4);
      if (lane < 4) {
        const int pp = blk * 8 + 2 * lane;
        sc[pp] = pp < n ? t0_ * 0.16f : -INFINITY;
        sc[pp + 1] = pp + 1 < n ? t1_ * 0.16f : -INFINITY;
      }
    }
    c1 = clock64();
    consumer_sync(nct);
    float mx = -INFINITY;
    for (int i = lane; i < n; i += 32) mx = fmaxf(mx, sc[i]);
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
    const float mn = fmaxf(am, mx);
    const float alpha = fast_exp2(am - mn);
#pragma unroll
    for (int k = 0; k < 4; ++k) dv[k] *= alpha;
    c2 = clock64();
    const int nk = (n + 15) >> 4;
    float lsum = 0.f;
    if (MODE == 0) {
      for (int j = 0; j < nk; ++j) {
        const int q0 = 16 * j + 2 * c;
        const float p0 = q0 < n ? fast_exp2(sc[q0] - mn) : 0.f;
        const float p1 = q0 + 1 < n ? fast_exp2(sc[q0 + 1] - mn) : 0.f;
        const float p2 = q0 + 8 < n ? fast_exp2(sc[q0 + 8] - mn) : 0.f;
        const float p3 = q0 + 9 < n ? fast_exp2(sc[q0 + 9] - mn) : 0.f;
        if (g == 0) lsum += (p0 + p1) + (p2 + p3);
        const uint32_t a0 = hilo(p0, p1, g), a2 = hilo(p2, p3, g);
        const int prow = 16 * j + (lane & 15);
        const uint32_t ra = Vb + prow * rowb;
        const int rot = (apos0 + prow) % nc;
        const uint32_t m0 = (q0 < n ? 0xffffu : 0u) | (q0 + 1 < n ? 0xffff0000u : 0u);
        const uint32_t m1 = (q0 + 8 < n ? 0xffffu : 0u) | (q0 + 9 < n ? 0xffff0000u : 0u);
        const int nb = warp;
        uint32_t b[2];
        ldsm_x2_trans(ra + (((nb + rot) % nc) * 16), b);
        mma_16816(dv, a0, a2, b[0] & m0, b[1] & m1);
      }
    } else {
      // variant: all exp2 / operands first (unrolled), then the MMA chain
      uint32_t A0[8], A2[8], B0[8], B1[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int q0 = 16 * j + 2 * c;
        float p0, p1, p2, p3;
        if (MODE == 2) {
          p0 = sc[q0] - mn; p1 = sc[q0 + 1] - mn; p2 = sc[q0 + 8] - mn; p3 = sc[q0 + 9] - mn;
        } else {
          p0 = fast_exp2(sc[q0] - mn); p1 = fast_exp2(sc[q0 + 1] - mn);
          p2 = fast_exp2(sc[q0 + 8] - mn); p3 = fast_exp2(sc[q0 + 9] - mn);
        }
        if (g == 0) lsum += (p0 + p1) + (p2 + p3);
        if (MODE == 3) {
          A0[j] = __float_as_uint(p0 + p1);
          A2[j] = __float_as_uint(p2 + p3);
        } else {
          A0[j] = hilo(p0, p1, g);
          A2[j] = hilo(p2, p3, g);
        }
        const int prow = 16 * j + (lane & 15);
        const int rot = (apos0 + prow) % nc;
        uint32_t b[2];
        if (MODE == 4) {
          b[0] = lane * j; b[1] = lane + j;
        } else {
          ldsm_x2_trans(Vb + prow * rowb + (((warp + rot) % nc) * 16), b);
        }
        B0[j] = b[0];
        B1[j] = b[1];
      }
      float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        if (MODE == 5) {
          dv[0] += __uint_as_float(A0[j] ^ B0[j]); e[1] += __uint_as_float(A2[j + 1] ^ B1[j + 1]);
        } else {
          mma_16816(dv, A0[j], A2[j], B0[j], B1[j]);
          mma_16816(e, A0[j + 1], A2[j + 1], B0[j + 1], B1[j + 1]);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) dv[k] += e[k];
    }
    for (int o2 = 1; o2 < 4; o2 <<= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o2);
    al = al * alpha + __shfl_sync(0xffffffffu, lsum, 0);
    am = mn;
    }
    const long long c3 = clock64();
    tsc += c1 - c0;
    tmax += c2 - c1;
    tpv += c3 - c2;
  }
  if (dv[0] + al == 12345.f) out[0] = dv[1];
  if (tid == 0) {
    cyc[blockIdx.x * 4 + 0] = (clock64() - t0) / nstages;
    cyc[blockIdx.x * 4 + 1] = tsc / nstages;
    cyc[blockIdx.x * 4 + 2] = tmax / nstages;
    cyc[blockIdx.x * 4 + 3] = tpv / nstages;
  }
}

template <int MODE>
void run() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 148 * 4 * 8);
  const int smem = 2 * kN * kD * 2 + 2 * kN * 4 + 2 * kN * 2;
  cudaFuncSetAttribute(att<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  att<MODE><<<148, 352, smem>>>(2000, out, cyc);
  cudaDeviceSynchronize();
  long long h[4];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("mode %d: %lld cycles/stage (scores %lld, sync+max %lld, P.V %lld) [%s]\n", MODE, h[0], h[1], h[2], h[3],
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>();
  run<1>();
  run<2>();
  run<3>();
  run<4>();
  run<5>();
  run<6>();
  run<7>();
  return 0;
}
