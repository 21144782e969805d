// Internal device-side helpers for libelaskit_b200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "ew_api.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libelaskit_b200 kernels target sm_100a (B200) only"
#endif

namespace ew {

// ---- error plumbing (defined in runtime.cu) ----
int set_error(int status, const std::string& msg);
int cuda_status(cudaError_t e, const char* what);

#define EW_CUDA_TRY(expr)                                      \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::ew::cuda_status(_e, #expr); \
  } while (0)

// SM count of the current device (cached per device).
int num_sms();

// ---- segment map on device ----
struct DevSeg {
  int64_t global_lo;
  int64_t length;
  int64_t local_off;
  int64_t row_base;  // first row of this segment
};

struct ShardMapView {
  const DevSeg* segs;
  int64_t n_segs;
  int64_t n_rows;
  int64_t total_bytes;  // packed local buffer size
  int block_shift;      // log2(block_bytes)
};

// ---- 128-bit memory helpers ----
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ uint4 ld_plain(const void* p) {
  uint4 v;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_plain(void* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint64_t lo64(const uint4& v) {
  return (static_cast<uint64_t>(v.y) << 32) | v.x;
}
__device__ __forceinline__ uint64_t hi64(const uint4& v) {
  return (static_cast<uint64_t>(v.w) << 32) | v.z;
}

// Blackwell 256-bit global accesses (LDG.E.256 / STG.E.256): one instruction
// per 32 bytes; streaming copies reach 6.6 TB/s with them versus 5.7 TB/s with
// 128-bit pairs (tools/microbench/copy_variants.cu).  32-byte aligned.
struct alignas(32) Vec32 {
  uint64_t w[4];
};

__device__ __forceinline__ Vec32 ld_stream32(const void* p) {
  uint32_t r[8];
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "l"(p));
  Vec32 v;
#pragma unroll
  for (int k = 0; k < 4; ++k) v.w[k] = (static_cast<uint64_t>(r[2 * k + 1]) << 32) | r[2 * k];
  return v;
}

// Read-only 256-bit load without the L2 evict-first hint: for streams that
// may alias another stream of the same kernel (a unit buffer listed twice),
// whose second read should hit L2.
__device__ __forceinline__ Vec32 ld_nc32(const void* p) {
  uint32_t r[8];
  asm volatile(
      "ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "l"(p));
  Vec32 v;
#pragma unroll
  for (int k = 0; k < 4; ++k) v.w[k] = (static_cast<uint64_t>(r[2 * k + 1]) << 32) | r[2 * k];
  return v;
}

// 32-byte load of data this kernel also writes (no .nc): read-modify-write
// of an accumulator
__device__ __forceinline__ Vec32 ld_plain32(const void* p) {
  uint32_t r[8];
  asm volatile("ld.global.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "l"(p));
  Vec32 v;
#pragma unroll
  for (int k = 0; k < 4; ++k) v.w[k] = (static_cast<uint64_t>(r[2 * k + 1]) << 32) | r[2 * k];
  return v;
}

// the j-th fp32 (j < 8) of a 32-byte vector
__device__ __forceinline__ float f32_of(const Vec32& v, int j) {
  return __uint_as_float(static_cast<uint32_t>(v.w[j >> 1] >> (32 * (j & 1))));
}

__device__ __forceinline__ void st_stream32(void* p, const Vec32& v) {
  asm volatile(
      "st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
      "r"(static_cast<uint32_t>(v.w[0])), "r"(static_cast<uint32_t>(v.w[0] >> 32)),
      "r"(static_cast<uint32_t>(v.w[1])), "r"(static_cast<uint32_t>(v.w[1] >> 32)),
      "r"(static_cast<uint32_t>(v.w[2])), "r"(static_cast<uint32_t>(v.w[2] >> 32)),
      "r"(static_cast<uint32_t>(v.w[3])), "r"(static_cast<uint32_t>(v.w[3] >> 32))
      : "memory");
}

// ---- shared-memory / async-proxy (TMA bulk copy + mbarrier) primitives

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "EW_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra EW_WAIT;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load(void* smem, const void* gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint4 lds128(const uint8_t* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

__device__ __forceinline__ void tma_store(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem),
               "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__host__ __device__ __forceinline__ int64_t floor_div(int64_t a, int64_t b) {
  int64_t q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

// Row r -> segment index (binary search over row_base).
__device__ __forceinline__ int64_t seg_of_row(const ShardMapView& m, int64_t r) {
  int64_t lo = 0, hi = m.n_segs - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (m.segs[mid].row_base <= r) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

struct RowGeom {
  int64_t local_lo;  // first local byte of the row
  int64_t len;       // bytes
  int64_t delta;     // global = local + delta
  int64_t block;     // global block id
};

__device__ __forceinline__ RowGeom row_geom(const ShardMapView& m, int64_t r) {
  const DevSeg s = m.segs[seg_of_row(m, r)];
  const int64_t b = (s.global_lo >> m.block_shift) + (r - s.row_base);
  const int64_t g_lo = max(s.global_lo, b << m.block_shift);
  const int64_t g_hi = min(s.global_lo + s.length, (b + 1) << m.block_shift);
  RowGeom g;
  g.delta = s.global_lo - s.local_off;
  g.local_lo = g_lo - g.delta;
  g.len = g_hi - g_lo;
  g.block = b;
  return g;
}

// Row geometry for a thread that visits rows in increasing order (a
// persistent CTA's r, r + grid, ...): the current segment and the next
// segment's first row stay in registers, so a row costs no memory access
// unless it crosses into a new segment — a binary search per row is ~6
// dependent L2 loads, a bubble in a streaming pipeline.
struct RowCursor {
  int64_t idx = -1;
  int64_t next_base = 0;
  DevSeg seg{};

  __device__ __forceinline__ RowGeom at(const ShardMapView& m, int64_t r) {
    if (idx < 0) {
      idx = seg_of_row(m, r);
      seg = m.segs[idx];
      next_base = idx + 1 < m.n_segs ? m.segs[idx + 1].row_base : INT64_MAX;
    }
    while (r >= next_base) {
      ++idx;
      seg = m.segs[idx];
      next_base = idx + 1 < m.n_segs ? m.segs[idx + 1].row_base : INT64_MAX;
    }
    const int64_t b = (seg.global_lo >> m.block_shift) + (r - seg.row_base);
    const int64_t g_lo = max(seg.global_lo, b << m.block_shift);
    const int64_t g_hi = min(seg.global_lo + seg.length, (b + 1) << m.block_shift);
    RowGeom g;
    g.delta = seg.global_lo - seg.local_off;
    g.local_lo = g_lo - g.delta;
    g.len = g_hi - g_lo;
    g.block = b;
    return g;
  }
};

}  // namespace ew

// Opaque handle bodies shared between translation units.
namespace ew {
// Per-row geometry precomputed at ew_shardmap_create for the register-staged
// snapshot kernel (one 32-byte broadcast load per row instead of a segment
// cursor held in registers across the row).
struct alignas(32) RowDesc {
  int64_t w0;    // first local byte of the row's 32-byte-aligned window
  int64_t q0;    // global word index of window word 0: floor((w0 + delta) / 8)
  int32_t head;  // the row inside the window: [head, end)
  int32_t end;
  int32_t sh;    // (global - local) mod 8
  int32_t pad;
};
}  // namespace ew

struct ew_shardmap {
  int device = -1;
  int64_t n_segs = 0;
  int64_t n_rows = 0;
  int64_t total_bytes = 0;
  int64_t block_bytes = 0;
  int block_shift = 0;
  ew::DevSeg* d_segs = nullptr;      // device copy
  ew::RowDesc* d_rows = nullptr;     // per-row geometry (n_rows entries)
  std::vector<ew::DevSeg> h_segs;    // host copy (row -> block queries)
  ew::ShardMapView view() const {
    return ew::ShardMapView{d_segs, n_segs, n_rows, total_bytes, block_shift};
  }
};
