// Microbenchmark: three formulations of the Philox-4x64 64x64->128 product on
// sm_100a (tools/microbench, not product code).  Prints G blocks/s for each.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define M0 0xD2E7470EE14C6C93ULL
#define M1 0xCA5A826395121157ULL

template <uint64_t A>
__device__ __forceinline__ void mul_v0(uint64_t b, uint64_t& hi, uint64_t& lo) {
  const uint32_t a0 = (uint32_t)A, a1 = (uint32_t)(A >> 32);
  const uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  uint64_t p00 = (uint64_t)a0 * b0;
  uint64_t p01 = (uint64_t)a0 * b1 + (p00 >> 32);
  uint64_t p10 = (uint64_t)a1 * b0 + (uint32_t)p01;
  uint64_t p11 = (uint64_t)a1 * b1 + (p01 >> 32);
  hi = p11 + (p10 >> 32);
  lo = ((uint64_t)(uint32_t)p10 << 32) | (uint32_t)p00;
}
template <uint64_t A>
__device__ __forceinline__ void mul_v1(uint64_t b, uint64_t& hi, uint64_t& lo) {
  hi = __umul64hi(A, b);
  lo = A * b;
}
template <uint64_t A>
__device__ __forceinline__ void mul_v2(uint64_t b, uint64_t& hi, uint64_t& lo) {
  const uint32_t a0 = (uint32_t)A, a1 = (uint32_t)(A >> 32);
  const uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  uint32_t r0, r1, r2, r3;
  asm("{\n\tmul.lo.u32 %0, %4, %6;\n\tmul.hi.u32 %1, %4, %6;\n\tmad.lo.cc.u32 %1, %4, %7, %1;\n\t"
      "madc.hi.u32 %2, %4, %7, 0;\n\tmad.lo.cc.u32 %1, %5, %6, %1;\n\tmadc.hi.cc.u32 %2, %5, %6, %2;\n\t"
      "madc.hi.u32 %3, %5, %7, 0;\n\tmad.lo.cc.u32 %2, %5, %7, %2;\n\taddc.u32 %3, %3, 0;\n\t}"
      : "=&r"(r0), "=&r"(r1), "=&r"(r2), "=&r"(r3) : "n"(a0), "n"(a1), "r"(b0), "r"(b1));
  lo = ((uint64_t)r1 << 32) | r0;
  hi = ((uint64_t)r3 << 32) | r2;
}

template <int V>
__global__ void kern(uint64_t seed, uint64_t lane, int64_t nblocks, uint64_t* sink) {
  uint64_t acc = 0;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblocks;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c0 = b + 1, c1 = 12345, c2 = lane, c3 = 0, k0 = seed, k1 = 0x454C41534B495431ULL;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      uint64_t h0, l0, h1, l1;
      if (V == 0) { mul_v0<M0>(c0, h0, l0); mul_v0<M1>(c2, h1, l1); }
      if (V == 1) { mul_v1<M0>(c0, h0, l0); mul_v1<M1>(c2, h1, l1); }
      if (V == 2) { mul_v2<M0>(c0, h0, l0); mul_v2<M1>(c2, h1, l1); }
      const uint64_t n0 = h1 ^ c1 ^ k0, n2 = h0 ^ c3 ^ k1;
      c0 = n0; c1 = l1; c2 = n2; c3 = l0;
      k0 += 0x9E3779B97F4A7C15ULL; k1 += 0xBB67AE8584CAA73BULL;
    }
    acc ^= c0 ^ c1 ^ c2 ^ c3;
  }
  if (acc == 0x1234567) sink[0] = acc;
}

int main() {
  uint64_t* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n = 1LL << 31;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (v == 0) kern<0><<<sms * 8, 256>>>(1, 7, n, sink);
      if (v == 1) kern<1><<<sms * 8, 256>>>(1, 7, n, sink);
      if (v == 2) kern<2><<<sms * 8, 256>>>(1, 7, n, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("variant %d: %.1f G blocks/s (%.2f ms)\n", v, n / ms / 1e6, ms);
    }
  }
  return 0;
}
