// (a) Per-step snapshot with fused per-block checksum, and verification.
//
// Replaces the reference's *modelled* snapshot (SnapshotTimeline /
// snapshot_overhead_s, param_fabric.hpp:86-96; Simulation::snapshot_delta,
// sim.cpp:861-880) with the byte-moving operation: one HBM pass copies a
// rank's packed shard live -> snapshot while checksumming it, a second pass
// re-reads the snapshot and compares.  Both are HBM-bound streaming kernels:
// a warp-specialised CTA streams its rows through a shared-memory ring with
// cp.async.bulk (TMA) loads and stores, one checksum row (<= 64 KiB) per CTA
// iteration, persistent grid of SMs x resident CTAs.
//
// Checksum spec (ew_api.h, oracle/ew_oracle.c ew_oracle_row_sums): per global
// block b, s0 = sum w_i and s1 = sum (i+1) w_i (mod 2^64) over the global
// little-endian u64 words w_i, bytes the buffer does not hold read as zero.
//
// Per local 8-byte word W at local byte x (8-aligned) the global position is
// g = x + delta, q = floor(g/8), sh = g mod 8 (uniform per row).  W feeds
// word q with A = W << 8sh and word q+1 with B = W >> (64-8sh) (sh > 0), so
// with C = A + B:  s0 += C,  s1 += (q+1) C + B.  Bytes outside the row are
// masked before the split, hence every nonzero contribution lands in the
// row's own block.  Per thread the word indices are q_t + 256 i (+1 for the
// odd word), so s1 needs only additions: sum i*D_i = n*T1 - T2 with the
// running sums T1 += D_i, T2 += T1 (D_i = C_even + C_odd of iteration i).
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
// TMA-fed variant: the load pipeline never drains at row boundaries.
//
// Warp 0 (one lane) streams 16 KiB pieces of this CTA's rows into a ring of
// shared-memory stages with cp.async.bulk (mbarrier complete_tx); four
// consumer warps checksum each stage from shared memory (16-byte units,
// conflict-free), the first consumer lane writes the snapshot copy of the
// stage back with one bulk shared->global store, and the stage is released
// once both the consumers and the store engine have read it.  Row sums are
// reduced through shared-memory slots (each consumer warp adds its sums, the
// last to arrive finishes the row), so neither the producer nor any consumer
// waits at a row end.  Unit k of a row's 32-byte-aligned window holds global
// words q_t + 256*i (+1 for the odd word), i = the thread's iteration.
constexpr int kTmaConsumers = 4;                  // warps
constexpr int kTmaThreads = 32 * (kTmaConsumers + 1);
constexpr int kTmaStages = 4;
constexpr int kTmaPiece = 16 * 1024;              // bytes per stage
constexpr int kTmaSmem = kTmaStages * kTmaPiece;  // 64 KiB -> 3 CTAs per SM
constexpr int kTmaUnitsPerThread = kTmaPiece / 16 / (32 * kTmaConsumers);  // 8

constexpr int kRowSlots = 8;                     // >= kTmaStages + 1, power of 2
static_assert(kRowSlots > kTmaStages, "row slots must cover the ring");

struct TmaRow {
  int64_t w0;      // first local byte of the 32-byte-aligned window
  int head, end;   // the row inside the window: [head, end)
  int n_pieces;
  int64_t window_bytes;
};

__device__ __forceinline__ TmaRow tma_row(const ShardMapView& m, int64_t r, RowGeom& g,
                                          RowCursor& cur) {
  g = cur.at(m, r);
  TmaRow t;
  t.w0 = g.local_lo & ~int64_t{31};
  t.head = static_cast<int>(g.local_lo - t.w0);
  t.end = t.head + static_cast<int>(g.len);
  t.window_bytes = ((g.local_lo + g.len + 31) & ~int64_t{31}) - t.w0;
  t.n_pieces = static_cast<int>((t.window_bytes + kTmaPiece - 1) / kTmaPiece);
  return t;
}

template <Mode M>
__global__ void __launch_bounds__(kTmaThreads, 3) tma_row_kernel(ShardMapView map,
                                                              const uint8_t* __restrict__ src,
                                                              uint8_t* __restrict__ dst,
                                                              uint64_t* __restrict__ row_sums,
                                                              const uint64_t* __restrict__ expected,
                                                              uint32_t* __restrict__ bad_count,
                                                              int64_t* __restrict__ bad_rows,
                                                              int64_t bad_cap) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kTmaStages];
  __shared__ __align__(8) uint64_t empty[kTmaStages];
  // per-row reduction slots: each consumer warp adds its sums, the last of
  // the four to arrive finishes the row (no consumer barrier, so no warp
  // ever waits for another at a row end).  A warp runs at most kTmaStages
  // pieces (so <= kTmaStages rows) ahead of the slowest: 8 slots suffice.
  __shared__ unsigned long long slot_s0[kRowSlots], slot_s1[kRowSlots];
  __shared__ unsigned slot_n[kRowSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < kRowSlots) {
    slot_s0[threadIdx.x] = 0;
    slot_s1[threadIdx.x] = 0;
    slot_n[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {  // producer
    if (lane != 0) return;
    RowCursor cur;
    int64_t k = 0;
    for (int64_t r = blockIdx.x; r < map.n_rows; r += gridDim.x) {
      RowGeom g;
      const TmaRow t = tma_row(map, r, g, cur);
      for (int p = 0; p < t.n_pieces; ++p, ++k) {
        const int s = static_cast<int>(k % kTmaStages);
        if (k >= kTmaStages) {
          mbar_wait(&empty[s], static_cast<uint32_t>(((k / kTmaStages) - 1) & 1));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const int64_t off = static_cast<int64_t>(p) * kTmaPiece;
        const uint32_t n =
            static_cast<uint32_t>(min(static_cast<int64_t>(kTmaPiece), t.window_bytes - off));
        mbar_expect_tx(&full[s], n);
        tma_load(ring + s * kTmaPiece, src + t.w0 + off, n, &full[s]);
      }
    }
    return;
  }

  const int ctid = threadIdx.x - 32;
  const int64_t last_vec_byte = (map.total_bytes - 1) & ~int64_t{31};  // start of the last 32-B vector
  const int partial = static_cast<int>(map.total_bytes & 31);
  int64_t k = 0;
  unsigned row_iter = 0;
  RowCursor cur;
  for (int64_t r = blockIdx.x; r < map.n_rows; r += gridDim.x) {
    RowGeom g;
    const TmaRow t = tma_row(map, r, g, cur);
    const int sh = static_cast<int>(g.delta & 7);
    const int64_t q_t = floor_div(t.w0 + 16 * ctid + g.delta, 8);
    uint64_t t1 = 0, t2 = 0, odd = 0, bsum = 0;
    for (int p = 0; p < t.n_pieces; ++p, ++k) {
      const int s = static_cast<int>(k % kTmaStages);
      mbar_wait(&full[s], static_cast<uint32_t>((k / kTmaStages) & 1));
      const uint8_t* stage = ring + s * kTmaPiece;
      const int base = p * kTmaPiece;  // window byte of the stage's first byte
      const int n = static_cast<int>(min(static_cast<int64_t>(kTmaPiece), t.window_bytes - base));
      if (M == Mode::kSnapshot && ctid == 0) {
        // store the 32-byte vectors this row owns (the row holding a
        // vector's first byte copies it); the buffer's partial last vector
        // goes through byte stores below
        int lo = (p == 0 && t.head != 0) ? 32 : 0;
        int hi = n;
        const int64_t last_in_window = last_vec_byte - t.w0 - base;
        if (partial && last_in_window >= 0 && last_in_window < n) hi = static_cast<int>(last_in_window);
        if (hi > lo) {
          tma_store(dst + t.w0 + base + lo, stage + lo, static_cast<uint32_t>(hi - lo));
          bulk_commit();
        }
      }
#pragma unroll
      for (int u = 0; u < kTmaUnitsPerThread; ++u) {
        const int x = 16 * (ctid + u * 32 * kTmaConsumers);  // byte in the stage
        const int wx = base + x;                             // byte in the window
        uint4 v = make_uint4(0, 0, 0, 0);
        if (x < n) v = lds128(stage + x);
        uint64_t w0 = lo64(v), w1 = hi64(v);
        if (wx < t.head || wx + 16 > t.end) {
          w0 &= byte_mask(wx, t.head, t.end);
          w1 &= byte_mask(wx + 8, t.head, t.end);
        }
        uint64_t c0 = w0, c1 = w1;
        if (sh != 0) {
          const uint64_t b0 = w0 >> (64 - 8 * sh), b1 = w1 >> (64 - 8 * sh);
          c0 = (w0 << (8 * sh)) + b0;
          c1 = (w1 << (8 * sh)) + b1;
          bsum += b0 + b1;
        }
        t1 += c0 + c1;
        t2 += t1;
        odd += c1;
      }
      if (M == Mode::kSnapshot && partial) {
        const int64_t last_in_window = last_vec_byte - t.w0 - base;
        if (last_in_window >= 0 && last_in_window < n && ctid < partial &&
            (last_in_window > 0 || p > 0 || t.head == 0))
          dst[t.w0 + base + last_in_window + ctid] = stage[last_in_window + ctid];
      }
      if (M == Mode::kSnapshot && ctid == 0) bulk_wait_read<0>();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    const int64_t n_exec = static_cast<int64_t>(t.n_pieces) * kTmaUnitsPerThread;
    uint64_t s0 = t1;
    uint64_t s1 = static_cast<uint64_t>(q_t + 1) * t1 +
                  static_cast<uint64_t>(2 * 32 * kTmaConsumers) *
                      (static_cast<uint64_t>(n_exec) * t1 - t2) + odd + bsum;
    s0 = warp_sum_u64(s0);
    s1 = warp_sum_u64(s1);
    const int sl = static_cast<int>(row_iter++ & (kRowSlots - 1));
    bool last = false;
    uint64_t x0 = 0, x1 = 0;
    if (lane == 0) {
      atomicAdd(&slot_s0[sl], static_cast<unsigned long long>(s0));
      atomicAdd(&slot_s1[sl], static_cast<unsigned long long>(s1));
      __threadfence_block();
      last = atomicAdd(&slot_n[sl], 1u) == kTmaConsumers - 1;
      if (last) {
        __threadfence_block();
        x0 = atomicExch(&slot_s0[sl], 0ull);
        x1 = atomicExch(&slot_s1[sl], 0ull);
        atomicExch(&slot_n[sl], 0u);
      }
    }
    if (last) {
      if (M == Mode::kVerify) {
        if (x0 != expected[2 * r] || x1 != expected[2 * r + 1]) {
          const uint32_t slot = atomicAdd(bad_count, 1u);
          if (bad_rows != nullptr && static_cast<int64_t>(slot) < bad_cap) bad_rows[slot] = r;
        }
      } else {
        row_sums[2 * r] = x0;
        row_sums[2 * r + 1] = x1;
      }
    }
  }
  if (M == Mode::kSnapshot && ctid == 0) bulk_wait_all();
}

template <Mode M>
int launch_rows(const ShardMapView& v, const uint8_t* src, uint8_t* dst, uint64_t* rows,
                const uint64_t* expected, uint32_t* bad, int64_t* bad_rows, int64_t cap,
                cudaStream_t stream) {
  auto k = tma_row_kernel<M>;
  // per device and cheap: set on every launch rather than caching
  EW_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kTmaThreads, kTmaSmem);
  const int64_t grid = std::min<int64_t>(v.n_rows, static_cast<int64_t>(num_sms()) * std::max(1, per_sm));
  k<<<static_cast<int>(grid), kTmaThreads, kTmaSmem, stream>>>(v, src, dst, rows, expected, bad,
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
  cudaError_t e = cudaGetDevice(&m->device);
  if (e == cudaSuccess && !dev.empty()) {
    e = cudaMalloc(&m->d_segs, dev.size() * sizeof(DevSeg));
    if (e == cudaSuccess)
      e = cudaMemcpy(m->d_segs, dev.data(), dev.size() * sizeof(DevSeg), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    if (m->d_segs) cudaFree(m->d_segs);
    delete m;
    return cuda_status(e, "ew_shardmap_create");
  }
  *out = m;
  return EW_OK;
}

void ew_shardmap_free(ew_shardmap* map) {
  if (map == nullptr) return;
  if (map->d_segs) cudaFree(map->d_segs);
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
  return launch_rows<Mode::kSnapshot>(map->view(), static_cast<const uint8_t*>(live),
                                      static_cast<uint8_t*>(snap), row_sums, nullptr, nullptr,
                                      nullptr, 0, (cudaStream_t)stream);
}

int ew_checksum(const ew_shardmap* map, const void* buf, uint64_t* row_sums,
                ew_stream_t stream) {
  if (map == nullptr || row_sums == nullptr || (map->total_bytes > 0 && !buf))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_checksum: NULL argument");
  if (!aligned32(buf)) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_checksum: buf must be 32-byte aligned");
  if (map->n_rows == 0) return EW_OK;
  return launch_rows<Mode::kChecksum>(map->view(), static_cast<const uint8_t*>(buf), nullptr,
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
  return launch_rows<Mode::kVerify>(map->view(), static_cast<const uint8_t*>(buf), nullptr,
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
