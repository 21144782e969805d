// (a) Per-step snapshot with fused per-block checksum, and verification.
//
// Replaces the reference's *modelled* snapshot (SnapshotTimeline /
// snapshot_overhead_s, param_fabric.hpp:86-96; Simulation::snapshot_delta,
// sim.cpp:861-880) with the byte-moving operation: one HBM pass copies a
// rank's packed shard live -> snapshot while checksumming it, a second pass
// re-reads the snapshot and compares.  Both are HBM-bound streaming kernels:
// one warp per checksum row (<= one block), 256-bit loads kept in registers,
// row sums reduced with shuffles (warp_row_kernel below).
//
// Checksum spec (ew_api.h, oracle/ew_oracle.c ew_oracle_row_sums,
// oracle/checksum_spec.py): per global block b, s0 = sum w_i and
// s1 = sum (i+1) w_i (mod 2^64) over the global little-endian u64 words w_i,
// bytes the buffer does not hold read as zero.
//
// Per local 8-byte word W at local byte x (8-aligned) the global position is
// g = x + delta, q = floor(g/8), sh = g mod 8 (uniform per row).  W feeds
// word q with A = W << 8sh and word q+1 with B = W >> (64-8sh) (sh > 0), so
// with C = A + B:  s0 += C,  s1 += (q+1) C + B.  Bytes outside the row are
// masked before the split, hence every nonzero contribution lands in the
// row's own block.
#include <algorithm>
#include <string>
#include <vector>

#include "ew_device.cuh"

namespace ew {
namespace {

__device__ __forceinline__ uint64_t byte_mask(int x, int a, int e) {
  // bytes of the 8-byte word at row-relative x that fall in [a, e)
  const int lo = min(max(a - x, 0), 8);
  const int hi = min(max(e - x, 0), 8);
  if (hi <= lo) return 0;
  const uint64_t upper = (hi == 8) ? ~0ULL : ((1ULL << (8 * hi)) - 1);
  return upper & (~0ULL << (8 * lo));
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

enum class Mode { kSnapshot, kChecksum, kVerify };

__global__ void rows_to_blocks_kernel(ShardMapView map, const uint64_t* __restrict__ rows,
                                      unsigned long long* __restrict__ blocks, int64_t n_blocks) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < map.n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const RowGeom g = row_geom(map, r);
    if (g.block < 0 || g.block >= n_blocks) continue;
    atomicAdd(&blocks[2 * g.block], static_cast<unsigned long long>(rows[2 * r]));
    atomicAdd(&blocks[2 * g.block + 1], static_cast<unsigned long long>(rows[2 * r + 1]));
  }
}

// Segment holding local byte x (binary search over local_off).
__device__ __forceinline__ int64_t seg_of_local(const ShardMapView& m, int64_t x) {
  int64_t lo = 0, hi = m.n_segs - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (m.segs[mid].local_off <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint8_t synth_byte(uint64_t seed, int64_t g) {
  return static_cast<uint8_t>(splitmix64(seed ^ static_cast<uint64_t>(g >> 3)) >> (8 * (g & 7)));
}

__global__ void fill_kernel(ShardMapView map, uint8_t* __restrict__ buf, uint64_t seed) {
  const int64_t nvec = (map.total_bytes + 15) >> 4;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = 16 * v;
    const DevSeg s = map.segs[seg_of_local(map, x)];
    const bool inside = x + 16 <= s.local_off + s.length && x + 16 <= map.total_bytes;
    if (inside) {
      const int64_t g = x + (s.global_lo - s.local_off);
      const int64_t q = g >> 3;
      const int sh = static_cast<int>(g & 7);
      const uint64_t w0 = splitmix64(seed ^ static_cast<uint64_t>(q));
      const uint64_t w1 = splitmix64(seed ^ static_cast<uint64_t>(q + 1));
      uint64_t lo, hi;
      if (sh == 0) {
        lo = w0;
        hi = w1;
      } else {
        const uint64_t w2 = splitmix64(seed ^ static_cast<uint64_t>(q + 2));
        lo = (w0 >> (8 * sh)) | (w1 << (64 - 8 * sh));
        hi = (w1 >> (8 * sh)) | (w2 << (64 - 8 * sh));
      }
      st_plain(buf + x, make_uint4(static_cast<uint32_t>(lo), static_cast<uint32_t>(lo >> 32),
                                   static_cast<uint32_t>(hi), static_cast<uint32_t>(hi >> 32)));
    } else {
      for (int k = 0; k < 16 && x + k < map.total_bytes; ++k) {
        const DevSeg t = map.segs[seg_of_local(map, x + k)];
        buf[x + k] = synth_byte(seed, x + k + (t.global_lo - t.local_off));
      }
    }
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; }

// ------------------------------------------------------------------------
// Register-staged variant (round 2): one WARP owns a row at a time.  Lanes
// stride 32 bytes through the row's 32-byte-aligned window with
// kWarpRowUnroll 256-bit loads in flight each, checksum in registers, store
// the snapshot copy straight back (STG.256), and reduce s0/s1 with shuffles
// at the row's end only.  No CTA barrier and no shared memory: no warp ever
// waits for another, so the load pipeline never drains (a CTA-wide row
// reduction capped register variants at 6.2-6.3 TB/s, the TMA ring at 6.45;
// this form measured 6.51-6.53 TB/s, tools/microbench/warp_row_variants.cu).
//
// Window word m (local byte w0 + 8m) is global word q0 + m with
// q0 = floor((w0 + delta) / 8), so with C_m and B_m as above
//     s0 = sum C_m,   s1 = (q0 + 1) s0 + sum m C_m + sum B_m,
// and per 32-byte vector j (words 4j..4j+3, c = C_0 + .. + C_3):
//     sum m C_m = 4 j c + (C_1 + 2 C_2 + 3 C_3).
// Copy ownership as in the ring kernel: a row stores the vectors whose first
// byte it holds; the buffer's partial last vector is stored bytewise.
constexpr int kWarpRowThreads = 256;        // per CTA
constexpr int kWarpRowUnroll = 4;           // 32-byte loads in flight per lane
constexpr int kWarpRowMinBlocks = 5;        // register cap: CTAs resident per SM
constexpr int kWarpRowGridPct = 160;        // grid = resident CTAs x this / 100
constexpr int kWarpRowStagger = 5;          // chunk rotation per warp (0: none)

template <Mode M>
__global__ void __launch_bounds__(kWarpRowThreads, kWarpRowMinBlocks) warp_row_kernel(
    const RowDesc* __restrict__ rows_desc, int n_rows, int64_t total_bytes,
    const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t* __restrict__ row_sums,
    const uint64_t* __restrict__ expected, uint32_t* __restrict__ bad_count,
    int64_t* __restrict__ bad_rows, int64_t bad_cap) {
  const int lane = threadIdx.x & 31;
  const int warp = static_cast<int>((blockIdx.x * kWarpRowThreads + threadIdx.x) >> 5);
  const int n_warps = static_cast<int>((gridDim.x * kWarpRowThreads) >> 5);
  for (int r = warp; r < n_rows; r += n_warps) {
    const RowDesc d = rows_desc[r];
    const Vec32* s = reinterpret_cast<const Vec32*>(src + d.w0);
    uint64_t s0 = 0, sj = 0, e = 0;
    auto accumulate = [&](const Vec32& v, int j) {
      const uint64_t cs = v.w[0] + v.w[1] + v.w[2] + v.w[3];
      s0 += cs;
      sj += static_cast<uint64_t>(j) * cs;
      e += v.w[1] + 2 * v.w[2] + 3 * v.w[3];
    };
    if (d.head == 0 && d.sh == 0 && (d.end & 31) == 0 &&
        (M != Mode::kSnapshot || d.w0 + d.end <= total_bytes)) {
      // fast path (every full, aligned row): no masks, no shifts, no
      // ownership or tail checks; kWarpRowUnroll loads in flight per lane
      const int nvec = d.end >> 5;
      // warps start their rows at staggered chunks (rotation by warp id):
      // in lockstep at the same offset, concurrent warps' addresses would
      // sit at a 64 KiB stride
      constexpr int kChunk = 32 * kWarpRowUnroll;
      const int n_chunks = (nvec + kChunk - 1) / kChunk;
      const int rot = (warp * kWarpRowStagger) % n_chunks;
      for (int c = 0; c < n_chunks; ++c) {
        int cc = c + rot;
        if (cc >= n_chunks) cc -= n_chunks;
        const int j0 = cc * kChunk + lane;
        Vec32 v[kWarpRowUnroll];
#pragma unroll
        for (int u = 0; u < kWarpRowUnroll; ++u) {
          const int j = j0 + 32 * u;
          v[u] = j < nvec ? ld_stream32(s + j) : Vec32{{0, 0, 0, 0}};
        }
#pragma unroll
        for (int u = 0; u < kWarpRowUnroll; ++u) {
          const int j = j0 + 32 * u;
          if (M == Mode::kSnapshot && j < nvec) st_stream32(dst + d.w0 + 32 * static_cast<int64_t>(j), v[u]);
          accumulate(v[u], j);  // zero vectors past the end add nothing
        }
      }
    } else {
      // general path (rows at segment edges: partial windows, realignment,
      // the buffer's last vector): one vector at a time
      const int nvec = (d.end + 31) >> 5;
      for (int j = lane; j < nvec; j += 32) {
        Vec32 v = ld_stream32(s + j);
        if (M == Mode::kSnapshot && !(j == 0 && d.head != 0)) {
          const int64_t x = d.w0 + 32 * static_cast<int64_t>(j);
          if (x + 32 <= total_bytes) {
            st_stream32(dst + x, v);
          } else {  // the buffer's partial last vector, once per buffer
#pragma unroll
            for (int k = 0; k < 31; ++k)
              if (x + k < total_bytes) dst[x + k] = static_cast<uint8_t>(v.w[k >> 3] >> (8 * (k & 7)));
          }
        }
        if (32 * j < d.head || 32 * j + 32 > d.end) {
#pragma unroll
          for (int k = 0; k < 4; ++k) v.w[k] &= byte_mask(32 * j + 8 * k, d.head, d.end);
        }
        if (d.sh != 0) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t b = v.w[k] >> (64 - 8 * d.sh);
            v.w[k] = (v.w[k] << (8 * d.sh)) + b;
            e += b;
          }
        }
        accumulate(v, j);
      }
    }
    uint64_t s1 = static_cast<uint64_t>(d.q0 + 1) * s0 + 4 * sj + e;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) {
      if (M == Mode::kVerify) {
        if (s0 != expected[2 * r] || s1 != expected[2 * r + 1]) {
          const uint32_t slot = atomicAdd(bad_count, 1u);
          if (bad_rows != nullptr && static_cast<int64_t>(slot) < bad_cap) bad_rows[slot] = r;
        }
      } else {
        row_sums[2 * r] = s0;
        row_sums[2 * r + 1] = s1;
      }
    }
  }
}

template <Mode M>
int launch_rows(const ew_shardmap* map, const uint8_t* src, uint8_t* dst, uint64_t* rows,
                const uint64_t* expected, uint32_t* bad, int64_t* bad_rows, int64_t cap,
                cudaStream_t stream) {
  // persistent: exactly the resident CTAs, warps take rows round-robin (a
  // second wave of CTAs would run its rows at low occupancy: a tail)
  auto k = warp_row_kernel<M>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kWarpRowThreads, 0);
  // balanced: every warp gets k or k - 1 rows (k = rows per warp at the
  // grid's capacity), so no last round runs with a fraction of the warps
  const int64_t warps_per_cta = kWarpRowThreads / 32;
  const int64_t cap_warps = std::max<int64_t>(
      1, static_cast<int64_t>(num_sms()) * std::max(1, per_sm) * kWarpRowGridPct / 100 * warps_per_cta);
  const int64_t k_rows = (map->n_rows + cap_warps - 1) / cap_warps;
  const int64_t n_warps = (map->n_rows + k_rows - 1) / k_rows;
  const int64_t grid = (n_warps + warps_per_cta - 1) / warps_per_cta;
  k<<<static_cast<int>(grid), kWarpRowThreads, 0, stream>>>(
      map->d_rows, static_cast<int>(map->n_rows), map->total_bytes, src, dst, rows, expected, bad,
      bad_rows, cap);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

}  // namespace
}  // namespace ew

using namespace ew;

extern "C" {

int ew_shardmap_create(const ew_segment* segs, int64_t n_segs, int64_t block_bytes,
                       ew_shardmap** out) {
  if (out == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n_segs < 0 || (n_segs > 0 && segs == nullptr))
    return set_error(EW_ERR_INVALID_ARGUMENT, "bad segment list");
  if (block_bytes < 4096 || block_bytes > (1 << 20) || (block_bytes & (block_bytes - 1)))
    return set_error(EW_ERR_INVALID_ARGUMENT, "block_bytes must be a power of two in [4 KiB, 1 MiB]");
  int shift = 0;
  while ((int64_t{1} << shift) < block_bytes) ++shift;

  auto* m = new ew_shardmap();
  m->block_bytes = block_bytes;
  m->block_shift = shift;
  int64_t local = 0, prev_hi = INT64_MIN, rows = 0;
  for (int64_t k = 0; k < n_segs; ++k) {
    const ew_segment& s = segs[k];
    if (s.length < 0 || s.global_lo < 0 || s.local_off != local || s.global_lo < prev_hi ||
        s.global_lo < s.local_off) {
      delete m;
      return set_error(EW_ERR_COVERAGE_MISMATCH,
                       "segments must be ascending, disjoint and packed back to back (segment " +
                           std::to_string(k) + ")");
    }
    DevSeg d{s.global_lo, s.length, s.local_off, rows};
    if (s.length > 0) rows += ((s.global_lo + s.length - 1) >> shift) - (s.global_lo >> shift) + 1;
    m->h_segs.push_back(d);
    local += s.length;
    prev_hi = s.global_lo + s.length;
  }
  // drop empty segments from the device table (they own no rows)
  std::vector<DevSeg> dev;
  for (const DevSeg& d : m->h_segs)
    if (d.length > 0) dev.push_back(d);
  m->h_segs = dev;
  m->n_segs = static_cast<int64_t>(dev.size());
  m->n_rows = rows;
  m->total_bytes = local;
  if (rows > INT32_MAX) {
    delete m;
    return set_error(EW_ERR_INVALID_ARGUMENT, "more than 2^31 rows: use larger blocks");
  }
  // per-row geometry for the snapshot / checksum / verify kernel
  std::vector<RowDesc> desc;
  desc.reserve(static_cast<size_t>(rows));
  for (const DevSeg& d : dev) {
    const int64_t delta = d.global_lo - d.local_off;
    const int64_t b0 = d.global_lo >> shift, b1 = (d.global_lo + d.length - 1) >> shift;
    for (int64_t b = b0; b <= b1; ++b) {
      const int64_t g_lo = std::max(d.global_lo, b << shift);
      const int64_t g_hi = std::min(d.global_lo + d.length, (b + 1) << shift);
      const int64_t local_lo = g_lo - delta;
      RowDesc r{};
      r.w0 = local_lo & ~int64_t{31};
      r.q0 = floor_div(r.w0 + delta, 8);
      r.head = static_cast<int32_t>(local_lo - r.w0);
      r.end = r.head + static_cast<int32_t>(g_hi - g_lo);
      r.sh = static_cast<int32_t>(delta & 7);
      desc.push_back(r);
    }
  }
  cudaError_t e = cudaGetDevice(&m->device);
  if (e == cudaSuccess && !dev.empty()) {
    e = cudaMalloc(&m->d_segs, dev.size() * sizeof(DevSeg));
    if (e == cudaSuccess)
      e = cudaMemcpy(m->d_segs, dev.data(), dev.size() * sizeof(DevSeg), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&m->d_rows, desc.size() * sizeof(RowDesc));
    if (e == cudaSuccess)
      e = cudaMemcpy(m->d_rows, desc.data(), desc.size() * sizeof(RowDesc), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    if (m->d_segs) cudaFree(m->d_segs);
    if (m->d_rows) cudaFree(m->d_rows);
    delete m;
    return cuda_status(e, "ew_shardmap_create");
  }
  *out = m;
  return EW_OK;
}

void ew_shardmap_free(ew_shardmap* map) {
  if (map == nullptr) return;
  if (map->d_segs) cudaFree(map->d_segs);
  if (map->d_rows) cudaFree(map->d_rows);
  delete map;
}

int64_t ew_shardmap_bytes(const ew_shardmap* map) { return map ? map->total_bytes : -1; }
int64_t ew_shardmap_num_rows(const ew_shardmap* map) { return map ? map->n_rows : -1; }

int ew_shardmap_row_blocks(const ew_shardmap* map, int64_t* out, int64_t cap) {
  if (map == nullptr || (out == nullptr && cap > 0))
    return set_error(EW_ERR_INVALID_ARGUMENT, "bad arguments");
  if (cap < map->n_rows) return set_error(EW_ERR_CAPACITY, "row block buffer too small");
  int64_t r = 0;
  for (const DevSeg& s : map->h_segs) {
    const int64_t b0 = s.global_lo >> map->block_shift;
    const int64_t b1 = (s.global_lo + s.length - 1) >> map->block_shift;
    for (int64_t b = b0; b <= b1; ++b) out[r++] = b;
  }
  return EW_OK;
}

int ew_snapshot(const ew_shardmap* map, const void* live, void* snap, uint64_t* row_sums,
                ew_stream_t stream) {
  if (map == nullptr || row_sums == nullptr || (map->total_bytes > 0 && (!live || !snap)))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_snapshot: NULL argument");
  if (!aligned32(live) || !aligned32(snap))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_snapshot: live/snap must be 32-byte aligned");
  if (map->n_rows == 0) return EW_OK;
  return launch_rows<Mode::kSnapshot>(map, static_cast<const uint8_t*>(live),
                                      static_cast<uint8_t*>(snap), row_sums, nullptr, nullptr,
                                      nullptr, 0, (cudaStream_t)stream);
}

int ew_checksum(const ew_shardmap* map, const void* buf, uint64_t* row_sums,
                ew_stream_t stream) {
  if (map == nullptr || row_sums == nullptr || (map->total_bytes > 0 && !buf))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_checksum: NULL argument");
  if (!aligned32(buf)) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_checksum: buf must be 32-byte aligned");
  if (map->n_rows == 0) return EW_OK;
  return launch_rows<Mode::kChecksum>(map, static_cast<const uint8_t*>(buf), nullptr,
                                      row_sums, nullptr, nullptr, nullptr, 0,
                                      (cudaStream_t)stream);
}

int ew_verify(const ew_shardmap* map, const void* buf, const uint64_t* expected,
              uint32_t* bad_count, int64_t* bad_rows, int64_t bad_cap, ew_stream_t stream) {
  if (map == nullptr || expected == nullptr || bad_count == nullptr ||
      (map->total_bytes > 0 && !buf))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_verify: NULL argument");
  if (!aligned32(buf)) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_verify: buf must be 32-byte aligned");
  EW_CUDA_TRY(cudaMemsetAsync(bad_count, 0, sizeof(uint32_t), (cudaStream_t)stream));
  if (map->n_rows == 0) return EW_OK;
  return launch_rows<Mode::kVerify>(map, static_cast<const uint8_t*>(buf), nullptr,
                                    nullptr, expected, bad_count, bad_rows, bad_cap,
                                    (cudaStream_t)stream);
}

int ew_rows_to_blocks(const ew_shardmap* map, const uint64_t* row_sums, uint64_t* block_sums,
                      int64_t n_blocks, ew_stream_t stream) {
  if (map == nullptr || row_sums == nullptr || block_sums == nullptr)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_rows_to_blocks: NULL argument");
  if (map->n_rows == 0) return EW_OK;
  const int grid = static_cast<int>(std::min<int64_t>((map->n_rows + 255) / 256, 4 * num_sms()));
  rows_to_blocks_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      map->view(), row_sums, reinterpret_cast<unsigned long long*>(block_sums), n_blocks);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

int ew_fill_synthetic(const ew_shardmap* map, void* buf, uint64_t seed, ew_stream_t stream) {
  if (map == nullptr || (map->total_bytes > 0 && buf == nullptr))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_fill_synthetic: NULL argument");
  if (!aligned16(buf)) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_fill_synthetic: buf must be 16-byte aligned");
  if (map->total_bytes == 0) return EW_OK;
  const int64_t nvec = (map->total_bytes + 15) >> 4;
  const int grid = static_cast<int>(std::min<int64_t>((nvec + 255) / 256, 8 * num_sms()));
  fill_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(map->view(), static_cast<uint8_t*>(buf),
                                                      seed);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

}  // extern "C"
