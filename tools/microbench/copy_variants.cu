// Microbenchmark: streaming-copy variants on sm_100a (tools only).  11.8 GB
// copy, grid-stride; 128-bit vs Blackwell 256-bit (.v8.b32) accesses and
// cache hints; prints TB/s (read+write bytes).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct alignas(32) v8 { uint32_t x[8]; };

template <int MODE, int U>
__global__ void __launch_bounds__(256) copyk(const v8* __restrict__ s, v8* __restrict__ d, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    v8 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        const v8* p = s + i;
        if (MODE == 0) {  // 2 x 128-bit, no_allocate
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x[0]), "=r"(v[u].x[1]), "=r"(v[u].x[2]), "=r"(v[u].x[3]) : "l"(p));
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x[4]), "=r"(v[u].x[5]), "=r"(v[u].x[6]), "=r"(v[u].x[7]) : "l"((const char*)p + 16));
        } else if (MODE == 1) {  // 256-bit
          asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(v[u].x[0]), "=r"(v[u].x[1]), "=r"(v[u].x[2]), "=r"(v[u].x[3]), "=r"(v[u].x[4]), "=r"(v[u].x[5]), "=r"(v[u].x[6]), "=r"(v[u].x[7]) : "l"(p));
        } else {  // 256-bit + L2 evict_first
          asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(v[u].x[0]), "=r"(v[u].x[1]), "=r"(v[u].x[2]), "=r"(v[u].x[3]), "=r"(v[u].x[4]), "=r"(v[u].x[5]), "=r"(v[u].x[6]), "=r"(v[u].x[7]) : "l"(p));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        v8* p = d + i;
        if (MODE == 0) {
          asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v[u].x[0]), "r"(v[u].x[1]), "r"(v[u].x[2]), "r"(v[u].x[3]) : "memory");
          asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"((char*)p + 16), "r"(v[u].x[4]), "r"(v[u].x[5]), "r"(v[u].x[6]), "r"(v[u].x[7]) : "memory");
        } else if (MODE == 1) {
          asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v[u].x[0]), "r"(v[u].x[1]), "r"(v[u].x[2]), "r"(v[u].x[3]), "r"(v[u].x[4]), "r"(v[u].x[5]), "r"(v[u].x[6]), "r"(v[u].x[7]) : "memory");
        } else {
          asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(v[u].x[0]), "r"(v[u].x[1]), "r"(v[u].x[2]), "r"(v[u].x[3]), "r"(v[u].x[4]), "r"(v[u].x[5]), "r"(v[u].x[6]), "r"(v[u].x[7]) : "memory");
        }
      }
    }
  }
}

template <int MODE, int U>
void run(const v8* s, v8* d, int64_t n, int grid, const char* name) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  copyk<MODE, U><<<grid, 256>>>(s, d, n);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    copyk<MODE, U><<<grid, 256>>>(s, d, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  printf("%-36s grid %5d: %.3f ms  %.2f TB/s\n", name, grid, best, 2.0 * n * 32 / best / 1e9);
}

int main() {
  const int64_t bytes = 11792227328LL, n = bytes / 32;
  v8 *s, *d;
  cudaMalloc(&s, bytes); cudaMalloc(&d, bytes);
  cudaMemset(s, 1, bytes); cudaMemset(d, 0, bytes);
  for (int grid : {148 * 4, 148 * 8}) {
    run<0, 2>(s, d, n, grid, "2x128-bit no_allocate U2");
    run<0, 4>(s, d, n, grid, "2x128-bit no_allocate U4");
    run<1, 2>(s, d, n, grid, "256-bit U2");
    run<1, 4>(s, d, n, grid, "256-bit U4");
    run<2, 2>(s, d, n, grid, "256-bit evict_first U2");
    run<2, 4>(s, d, n, grid, "256-bit evict_first U4");
  }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(a); cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  printf("%-36s            %.3f ms  %.2f TB/s\n", "cudaMemcpyAsync D2D", best, 2.0 * bytes / best / 1e9);
  return 0;
}
