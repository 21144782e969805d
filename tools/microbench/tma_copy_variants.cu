// Microbenchmark (tools only): where does the fused snapshot lose against a
// plain copy?  TMA ring copies of an 11.8 GB buffer (producer lane:
// cp.async.bulk global->shared; one consumer lane: bulk shared->global store),
// varying the piece order (each CTA owns 64 KiB rows, grid-stride over rows —
// the snapshot kernel's order — versus a dense sweep where consecutive CTAs
// take consecutive pieces), the checksum work of the consumers (none, or the
// snapshot's running sums over every 16-byte unit), ring depth and piece
// size.  Controls: 256-bit register grid-stride copy and cudaMemcpyAsync D2D.
// Prints TB/s (read + write bytes), best of 5.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tma_copy_variants tma_copy_variants.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma_load(void* s, const void* g, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(s)), "l"(g), "r"(n), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma_store(void* g, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(n) : "memory");
}
__device__ __forceinline__ uint4 lds128(const uint8_t* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
  return v;
}

constexpr int kConsumers = 4;
constexpr int kRow = 64 * 1024;

// ORDER 0: CTA owns rows r = blockIdx + k*grid, each row's pieces in order.
// ORDER 1: piece p = blockIdx + k*grid (dense sweep).
template <int ORDER, bool CHECK, int STAGES, int PIECE>
__global__ void __launch_bounds__(32 * (kConsumers + 1)) ring_copy(const uint8_t* __restrict__ src,
                                                                   uint8_t* __restrict__ dst,
                                                                   int64_t bytes,
                                                                   unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kConsumers); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t n_pieces = bytes / PIECE;  // tail ignored (bench sizes are multiples)
  constexpr int per_row = kRow / PIECE;
  const int64_t n_rows = n_pieces / per_row;
  // k-th piece of this CTA
  auto piece = [&](int64_t k) -> int64_t {
    if (ORDER == 1) return blockIdx.x + k * gridDim.x;
    const int64_t r = blockIdx.x + (k / per_row) * gridDim.x;
    return r * per_row + (k % per_row);
  };
  const int64_t mine = ORDER == 1 ? (n_pieces - blockIdx.x + gridDim.x - 1) / gridDim.x
                                  : ((n_rows - blockIdx.x + gridDim.x - 1) / gridDim.x) * per_row;
  if (warp == 0) {
    if (lane != 0) return;
    for (int64_t k = 0; k < mine; ++k) {
      const int s = k % STAGES;
      if (k >= STAGES) {
        mbar_wait(&empty[s], ((k / STAGES) - 1) & 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      mbar_expect_tx(&full[s], PIECE);
      tma_load(ring + s * PIECE, src + piece(k) * PIECE, PIECE, &full[s]);
    }
    return;
  }
  const int ctid = threadIdx.x - 32;
  uint64_t t1 = 0, t2 = 0;
  for (int64_t k = 0; k < mine; ++k) {
    const int s = k % STAGES;
    mbar_wait(&full[s], (k / STAGES) & 1);
    const uint8_t* st = ring + s * PIECE;
    if (ctid == 0) {
      tma_store(dst + piece(k) * PIECE, st, PIECE);
      asm volatile("cp.async.bulk.commit_group;");
    }
    if (CHECK) {
#pragma unroll
      for (int u = 0; u < PIECE / 16 / (32 * kConsumers); ++u) {
        const uint4 v = lds128(st + 16 * (ctid + u * 32 * kConsumers));
        const uint64_t w0 = (uint64_t(v.y) << 32) | v.x, w1 = (uint64_t(v.w) << 32) | v.z;
        t1 += w0 + w1;
        t2 += t1;
      }
    }
    if (ctid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (ctid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (CHECK && (t1 ^ t2) == 0x1234567ULL) atomicAdd(sink, 1ull);  // keep the sums live
}

struct alignas(32) v8 { uint32_t x[8]; };
__global__ void __launch_bounds__(256) reg_copy(const v8* __restrict__ s, v8* __restrict__ d, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
    v8 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n)
        asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(v[u].x[0]), "=r"(v[u].x[1]), "=r"(v[u].x[2]), "=r"(v[u].x[3]), "=r"(v[u].x[4]), "=r"(v[u].x[5]), "=r"(v[u].x[6]), "=r"(v[u].x[7]) : "l"(s + i));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n)
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(d + i), "r"(v[u].x[0]), "r"(v[u].x[1]), "r"(v[u].x[2]), "r"(v[u].x[3]), "r"(v[u].x[4]), "r"(v[u].x[5]), "r"(v[u].x[6]), "r"(v[u].x[7]) : "memory");
    }
  }
}

template <typename F>
float best_ms(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int sms;
unsigned long long* sink;

template <int ORDER, bool CHECK, int STAGES, int PIECE>
void ring(const uint8_t* s, uint8_t* d, int64_t bytes) {
  auto k = ring_copy<ORDER, CHECK, STAGES, PIECE>;
  const int smem = STAGES * PIECE;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * (kConsumers + 1), smem);
  const int grid = sms * per_sm;
  const float ms = best_ms([&] { k<<<grid, 32 * (kConsumers + 1), smem>>>(s, d, bytes, sink); });
  cudaError_t e = cudaGetLastError();
  printf("{\"kernel\": \"ring\", \"order\": \"%s\", \"checksum\": %d, \"stages\": %d, \"piece_kib\": %d, "
         "\"ctas_per_sm\": %d, \"ms\": %.3f, \"TBps\": %.3f%s}\n",
         ORDER ? "dense" : "rows", CHECK ? 1 : 0, STAGES, PIECE / 1024, per_sm, ms,
         2.0 * bytes / ms / 1e9, e == cudaSuccess ? "" : ", \"error\": 1");
}

int main() {
  const int64_t bytes = 11792400384LL;  // 7B rank shard rounded up to 64 KiB rows
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t *s, *d;
  cudaMalloc(&s, bytes); cudaMalloc(&d, bytes); cudaMalloc(&sink, 8);
  cudaMemset(s, 1, bytes); cudaMemset(d, 0, bytes);
  ring<0, false, 4, 16384>(s, d, bytes);
  ring<1, false, 4, 16384>(s, d, bytes);
  ring<0, true, 4, 16384>(s, d, bytes);
  ring<1, true, 4, 16384>(s, d, bytes);
  ring<0, false, 3, 16384>(s, d, bytes);
  ring<1, false, 3, 16384>(s, d, bytes);
  ring<1, false, 2, 32768>(s, d, bytes);
  ring<1, true, 2, 32768>(s, d, bytes);
  ring<1, false, 8, 8192>(s, d, bytes);
  ring<1, true, 8, 8192>(s, d, bytes);
  ring<1, false, 6, 8192>(s, d, bytes);
  ring<1, false, 2, 16384>(s, d, bytes);
  for (int g : {4, 8}) {
    const int grid = sms * g;
    const float ms = best_ms([&] { reg_copy<<<grid, 256>>>((const v8*)s, (v8*)d, bytes / 32); });
    printf("{\"kernel\": \"reg256\", \"grid\": %d, \"ms\": %.3f, \"TBps\": %.3f}\n", grid, ms, 2.0 * bytes / ms / 1e9);
  }
  const float ms = best_ms([&] { cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice); });
  printf("{\"kernel\": \"cudaMemcpyAsync\", \"ms\": %.3f, \"TBps\": %.3f}\n", ms, 2.0 * bytes / ms / 1e9);
  return 0;
}
