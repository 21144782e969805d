// Microbenchmark (tools only): can a register-staged snapshot (copy fused with
// the position-weighted block checksum) reach the plain-copy rate if no CTA
// barrier ever drains the load pipeline?  One WARP owns a 64 KiB block at a
// time (lanes stride 32 B through it, U loads in flight each), keeps s0 / s1
// in registers and reduces with shuffles at the block's end only.
// Aligned case (segment == whole buffer).  Controls: the 256-bit grid-stride
// copy and cudaMemcpyAsync.  Prints TB/s (read + write), best of 5, and checks
// the block sums against a scalar kernel.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o warp_row_variants warp_row_variants.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

struct alignas(32) V { uint64_t w[4]; };
__device__ __forceinline__ V ld32(const void* p) {
  uint32_t r[8];
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(p));
  V v; for (int k = 0; k < 4; ++k) v.w[k] = ((uint64_t)r[2 * k + 1] << 32) | r[2 * k]; return v;
}
__device__ __forceinline__ void st32(void* p, const V& v) {
  asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p),
               "r"((uint32_t)v.w[0]), "r"((uint32_t)(v.w[0] >> 32)), "r"((uint32_t)v.w[1]), "r"((uint32_t)(v.w[1] >> 32)),
               "r"((uint32_t)v.w[2]), "r"((uint32_t)(v.w[2] >> 32)), "r"((uint32_t)v.w[3]), "r"((uint32_t)(v.w[3] >> 32)) : "memory");
}

__global__ void copy256(const V* s, V* d, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += 2 * stride) {
    V a = ld32(s + i0), b;
    const bool two = i0 + stride < n;
    if (two) b = ld32(s + i0 + stride);
    st32(d + i0, a);
    if (two) st32(d + i0 + stride, b);
  }
}

// one warp per 64 KiB block; U 32-byte loads in flight per lane
template <int U, int T>
__global__ void __launch_bounds__(T) warp_rows(const uint8_t* s, uint8_t* d, int64_t nblocks, uint64_t* sums) {
  constexpr int kVec = 65536 / 32;  // 32-byte vectors per block
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)T + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * T) >> 5;
  for (int64_t b = wid; b < nblocks; b += nw) {
    const V* src = reinterpret_cast<const V*>(s + b * 65536);
    V* dst = reinterpret_cast<V*>(d + b * 65536);
    uint64_t s0 = 0, s1 = 0;
    const uint64_t word0 = (uint64_t)b * 8192;  // global word index of the block's first word
#pragma unroll 1
    for (int it = 0; it < kVec / 32; it += U) {
      V v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld32(src + (it + u) * 32 + lane);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        st32(dst + (it + u) * 32 + lane, v[u]);
        const uint64_t i1 = word0 + 4 * ((it + u) * 32 + lane) + 1;  // (i+1) of word 0
        const uint64_t c = v[u].w[0] + v[u].w[1] + v[u].w[2] + v[u].w[3];
        s0 += c;
        s1 += i1 * c + v[u].w[1] + 2 * v[u].w[2] + 3 * v[u].w[3];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) { sums[2 * b] = s0; sums[2 * b + 1] = s1; }
  }
}

__global__ void ref_sums(const uint64_t* w, int64_t nblocks, uint64_t* sums) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblocks; b += (int64_t)gridDim.x * blockDim.x) {
    uint64_t s0 = 0, s1 = 0;
    for (int64_t i = b * 8192; i < (b + 1) * 8192; ++i) { s0 += w[i]; s1 += (uint64_t)(i + 1) * w[i]; }
    sums[2 * b] = s0; sums[2 * b + 1] = s1;
  }
}
__global__ void fill(uint64_t* w, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i + 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; w[i] = z ^ (z >> 31);
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t bytes = 11792220160LL / 65536 * 65536, nblocks = bytes / 65536;
  uint8_t *s, *d; uint64_t *sums, *ref;
  cudaMalloc(&s, bytes); cudaMalloc(&d, bytes); cudaMalloc(&sums, nblocks * 16); cudaMalloc(&ref, nblocks * 16);
  fill<<<sms * 8, 256>>>((uint64_t*)s, bytes / 8);
  ref_sums<<<sms * 4, 128>>>((const uint64_t*)s, nblocks, ref);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto fn, bool check) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(sums, 0, nblocks * 16);
      cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    bool ok = true;
    if (check) {
      static uint64_t h1[2 * 200000], h2[2 * 200000];
      cudaMemcpy(h1, sums, nblocks * 16, cudaMemcpyDeviceToHost); cudaMemcpy(h2, ref, nblocks * 16, cudaMemcpyDeviceToHost);
      for (int64_t i = 0; i < 2 * nblocks; ++i) ok = ok && h1[i] == h2[i];
    }
    printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"TBps\": %.3f%s}\n", name, best, 2.0 * bytes / (best * 1e-3) / 1e12,
           check ? (ok ? ", \"sums\": \"ok\"" : ", \"sums\": \"MISMATCH\"") : "");
    if (cudaGetLastError() != cudaSuccess) printf("cuda error\n");
  };
  timeit("cudaMemcpyAsync", [&] { cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice); }, false);
  timeit("copy256 grid 8/SM", [&] { copy256<<<sms * 8, 256>>>((const V*)s, (V*)d, bytes / 32); }, false);
  timeit("warp_rows U4 T256 8/SM", [&] { warp_rows<4, 256><<<sms * 8, 256>>>(s, d, nblocks, sums); }, true);
  timeit("warp_rows U4 T256 6/SM", [&] { warp_rows<4, 256><<<sms * 6, 256>>>(s, d, nblocks, sums); }, true);
  timeit("warp_rows U8 T256 4/SM", [&] { warp_rows<8, 256><<<sms * 4, 256>>>(s, d, nblocks, sums); }, true);
  timeit("warp_rows U8 T256 6/SM", [&] { warp_rows<8, 256><<<sms * 6, 256>>>(s, d, nblocks, sums); }, true);
  timeit("warp_rows U2 T256 8/SM", [&] { warp_rows<2, 256><<<sms * 8, 256>>>(s, d, nblocks, sums); }, true);
  timeit("warp_rows U4 T128 16/SM", [&] { warp_rows<4, 128><<<sms * 16, 128>>>(s, d, nblocks, sums); }, true);
  return 0;
}
