// Microbenchmark: launch shapes of a row-per-CTA streaming copy+checksum
// (the snapshot kernel's structure) with 256-bit accesses (tools only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct alignas(32) V { uint64_t w[4]; };
__device__ __forceinline__ V ld32(const void* p) {
  uint32_t r[8];
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(p));
  V v; for (int k = 0; k < 4; ++k) v.w[k] = ((uint64_t)r[2*k+1] << 32) | r[2*k]; return v;
}
__device__ __forceinline__ void st32(void* p, const V& v) {
  asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p),
               "r"((uint32_t)v.w[0]), "r"((uint32_t)(v.w[0]>>32)), "r"((uint32_t)v.w[1]), "r"((uint32_t)(v.w[1]>>32)),
               "r"((uint32_t)v.w[2]), "r"((uint32_t)(v.w[2]>>32)), "r"((uint32_t)v.w[3]), "r"((uint32_t)(v.w[3]>>32)) : "memory");
}

template <int T, int U, int MINB, int ROW>
__global__ void __launch_bounds__(T, MINB) rowk(const uint8_t* s, uint8_t* d, int64_t nrows, uint64_t* out) {
  __shared__ uint64_t red[T / 32];
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int nvec = ROW / 32;
    const uint8_t* sv = s + r * ROW; uint8_t* dv = d + r * ROW;
    uint64_t t1 = 0, t2 = 0, odd = 0;
    for (int it = 0; it < (nvec + T - 1) / T; it += U) {
      V v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) { int idx = threadIdx.x + (it + u) * T; if (idx < nvec) v[u] = ld32(sv + 32 * idx); else v[u] = V{{0,0,0,0}}; }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int idx = threadIdx.x + (it + u) * T;
        if (idx < nvec) st32(dv + 32 * idx, v[u]);
        uint64_t c23 = v[u].w[2] + v[u].w[3];
        t1 += v[u].w[0] + v[u].w[1] + c23; t2 += t1; odd += v[u].w[1] + c23 + c23 + v[u].w[3];
      }
    }
    uint64_t s1 = t1 * 3 + t2 + odd;
    for (int o = 16; o > 0; o >>= 1) s1 += __shfl_down_sync(0xffffffffu, s1, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s1;
    __syncthreads();
    if (threadIdx.x == 0) { uint64_t x = 0; for (int w = 0; w < T / 32; ++w) x += red[w]; out[r] = x; }
    __syncthreads();
  }
}

template <int T, int U, int MINB, int ROW>
void run(const uint8_t* s, uint8_t* d, int64_t bytes, uint64_t* out, int sms) {
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rowk<T, U, MINB, ROW>, T, 0);
  int64_t nrows = bytes / ROW;
  int grid = (int)std::min<int64_t>(nrows, (int64_t)sms * per);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  rowk<T, U, MINB, ROW><<<grid, T>>>(s, d, nrows, out);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(a); rowk<T, U, MINB, ROW><<<grid, T>>>(s, d, nrows, out); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  printf("T %4d U %d minB %d row %6d occ %d grid %5d: %.3f ms %.2f TB/s\n", T, U, MINB, ROW, per, grid, best, 2.0 * nrows * ROW / best / 1e9);
}

template <int T, int U, int MINB>
__global__ void __launch_bounds__(T, MINB) flatk(const uint8_t* s, uint8_t* d, int64_t nchunks, uint64_t* out) {
  // chunk = T vectors of 32 B (8 KiB at T=256); CTA b takes chunks b + (i*U+u)*G
  __shared__ uint64_t red[U][T / 32];
  const int64_t G = gridDim.x;
  for (int64_t base = blockIdx.x; base < nchunks; base += (int64_t)U * G) {
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = base + u * G;
      if (c < nchunks) v[u] = ld32(s + (c * T + threadIdx.x) * 32); else v[u] = V{{0,0,0,0}};
    }
    uint64_t acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = base + u * G;
      if (c < nchunks) st32(d + (c * T + threadIdx.x) * 32, v[u]);
      uint64_t c23 = v[u].w[2] + v[u].w[3];
      acc[u] = v[u].w[0] + v[u].w[1] + c23 + (v[u].w[1] + c23 + c23 + v[u].w[3]) * 7;
      for (int o = 16; o > 0; o >>= 1) acc[u] += __shfl_down_sync(0xffffffffu, acc[u], o);
      if ((threadIdx.x & 31) == 0) red[u][threadIdx.x >> 5] = acc[u];
    }
    __syncthreads();
    if (threadIdx.x < U) {
      const int64_t c = base + threadIdx.x * G;
      uint64_t x = 0; for (int w = 0; w < T / 32; ++w) x += red[threadIdx.x][w];
      if (c < nchunks) out[c] = x;
    }
    __syncthreads();
  }
}

template <int T, int U, int MINB>
void runf(const uint8_t* s, uint8_t* d, int64_t bytes, uint64_t* out, int sms) {
  int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, flatk<T, U, MINB>, T, 0);
  int64_t nchunks = bytes / (T * 32);
  int grid = sms * per;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  flatk<T, U, MINB><<<grid, T>>>(s, d, nchunks, out);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(a); flatk<T, U, MINB><<<grid, T>>>(s, d, nchunks, out); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  printf("FLAT T %4d U %d minB %d occ %d grid %5d: %.3f ms %.2f TB/s\n", T, U, MINB, per, grid, best, 2.0 * nchunks * T * 32 / best / 1e9);
}

int main() {
  const int64_t bytes = 11792227328LL;
  uint8_t *s, *d; uint64_t* out;
  cudaMalloc(&s, bytes); cudaMalloc(&d, bytes); cudaMalloc(&out, bytes / 4096 * 8);
  cudaMemset(s, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  runf<256, 2, 4>(s, d, bytes, out, sms);
  runf<256, 4, 4>(s, d, bytes, out, sms);
  runf<256, 2, 8>(s, d, bytes, out, sms);
  runf<256, 4, 6>(s, d, bytes, out, sms);
  runf<512, 2, 4>(s, d, bytes, out, sms);
  run<256, 4, 4, 65536>(s, d, bytes, out, sms);
  run<256, 2, 4, 65536>(s, d, bytes, out, sms);
  run<256, 2, 6, 65536>(s, d, bytes, out, sms);
  run<256, 2, 8, 65536>(s, d, bytes, out, sms);
  run<128, 4, 8, 65536>(s, d, bytes, out, sms);
  run<128, 2, 12, 65536>(s, d, bytes, out, sms);
  run<512, 2, 2, 65536>(s, d, bytes, out, sms);
  run<512, 2, 3, 65536>(s, d, bytes, out, sms);
  run<256, 2, 8, 32768>(s, d, bytes, out, sms);
  run<256, 4, 4, 131072>(s, d, bytes, out, sms);
  return 0;
}
