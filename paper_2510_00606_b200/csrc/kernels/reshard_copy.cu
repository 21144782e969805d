// (b) Reshard executor: the planner's TransferPlan lowered to copies and run
// over NVLink/NVSwitch peer pointers plus local HBM.
//
// The reference only *times* a remap (remap_time, sim.cpp:452-483: max lane
// bytes / 25 GB/s).  Here each GPU executes its copy program (b200.hpp
// reshard_copies) in one launch: remote copies are 128-bit stores into
// IPC-mapped peer HBM (push) — or bulk loads from it (pull) — and local copies
// move retained bytes to their new packed position and the ring holder's
// self lanes.  The first CTAs take remote copies (NVLink-bound), the rest the
// local ones (HBM-bound).
//
// Each CTA is warp-specialised around a shared-memory ring:
//   producer (one elected lane): cp.async.bulk global -> shared of the
//     16-byte-aligned source window of each piece, completing on a per-stage
//     mbarrier — the Tensor Memory Accelerator keeps ~kStages x 16 KiB in
//     flight per CTA with no register traffic;
//   consumers (8 warps): read the stage, realign it to the destination when
//     source and destination are not congruent mod 16 (byte-granular plans,
//     SURVEY fact 9), write 16-byte vectors (or one bulk shared->global
//     store when congruent), and byte-store the partial vectors at copy ends
//     so adjacent copies from other GPUs never race on a vector; in a
//     verified program they also checksum what lands (kernel (a)'s spec,
//     labelled by NEW's segment map) while the bulk store drains; then
//     release the stage on its "empty" mbarrier.
// The producer resolves each piece (binary search over the items) once and
// passes the descriptor to the consumers in shared memory with the stage.
// Pieces are <= 16 KiB and cut at 16 KiB-aligned destination addresses, so
// no two pieces share a destination vector.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ew_device.cuh"

namespace ew {
namespace {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = 32 * (kConsumerWarps + 1);
constexpr int kStages = 6;
constexpr int kPiece = 16 * 1024;          // destination bytes per piece
// aligned source window of a piece (<= kPiece + 30) plus the realigning
// reader's 32-byte overhang
constexpr int kStageBytes = kPiece + 64;
constexpr int kSmem = kStages * kStageBytes;

struct CopyItem {
  const uint8_t* src;
  uint8_t* dst;
  int64_t bytes;
  int64_t piece_base;  // first piece id of this item within its class
  int64_t glob;        // global position of dst[0] (verified programs), else -1
  int64_t no_store;    // 1: checksum only (in-place retained bytes), no write
};

__host__ __device__ __forceinline__ int64_t pieces_of(const uint8_t* dst, int64_t bytes) {
  if (bytes <= 0) return 0;
  const uint64_t d = reinterpret_cast<uintptr_t>(dst);
  return static_cast<int64_t>((d + bytes - 1) / kPiece - d / kPiece + 1);
}

__device__ __forceinline__ int64_t item_of_piece(const CopyItem* items, int64_t n, int64_t p) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (items[mid].piece_base <= p) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

struct Piece {
  const uint8_t* src;  // first source byte
  uint8_t* dst;        // first destination byte
  int32_t bytes;
  bool no_store;
  int64_t glob;        // global position of dst[0], or -1
};

// The producer's pieces increase (first + k * step), so the item they fall
// in only moves forward: keep it and the next item's first piece in
// registers and touch the item list only when a piece crosses into a new
// item (a binary search per piece is ~log2(items) dependent L2 loads, a
// bubble in the producer's issue loop).
struct ItemCursor {
  int64_t idx = -1;
  int64_t next_base = 0;
  CopyItem it{};

  __device__ __forceinline__ const CopyItem& at(const CopyItem* list, int64_t n, int64_t p) {
    if (idx < 0) {
      idx = item_of_piece(list, n, p);
      it = list[idx];
      next_base = idx + 1 < n ? list[idx + 1].piece_base : INT64_MAX;
    }
    while (p >= next_base) {
      ++idx;
      it = list[idx];
      next_base = idx + 1 < n ? list[idx + 1].piece_base : INT64_MAX;
    }
    return it;
  }
};

__device__ __forceinline__ Piece piece_at(const CopyItem& it, int64_t p) {
  const uint64_t d = reinterpret_cast<uintptr_t>(it.dst);
  const uint64_t cut = (d / kPiece + static_cast<uint64_t>(p - it.piece_base)) * kPiece;
  const uint64_t lo = max(d, cut);
  const uint64_t hi = min(d + static_cast<uint64_t>(it.bytes), cut + kPiece);
  return Piece{it.src + (lo - d), it.dst + (lo - d), static_cast<int32_t>(hi - lo),
               it.no_store != 0,
               it.glob >= 0 ? it.glob + static_cast<int64_t>(lo - d) : int64_t{-1}};
}

// Verification on arrival: kernel (a)'s checksum (s0 = sum w, s1 = sum (i+1) w
// over global u64 words) of the bytes a piece lands, labelled with the
// global position of their destination, added to global block sums.  Warp w
// takes a contiguous quarter of the piece's words (<= 513 words, so at most
// two checksum blocks of >= 4 KiB), lanes stride by one word (conflict-free
// 8-byte shared loads), and lane 0 adds the warp's sums with <= 4 atomics.
// Warp sum mod 2^64 with the single-instruction 32-bit reduction (REDUX):
// four 16-bit limbs, each limb's 32-lane sum exact in 21 bits.
__device__ __forceinline__ uint64_t warp_sum64(uint64_t x) {
  const unsigned m = 0xffffffffu;
  const uint64_t l0 = __reduce_add_sync(m, static_cast<unsigned>(x & 0xffff));
  const uint64_t l1 = __reduce_add_sync(m, static_cast<unsigned>((x >> 16) & 0xffff));
  const uint64_t l2 = __reduce_add_sync(m, static_cast<unsigned>((x >> 32) & 0xffff));
  const uint64_t l3 = __reduce_add_sync(m, static_cast<unsigned>(x >> 48));
  return l0 + (l1 << 16) + (l2 << 32) + (l3 << 48);
}

__device__ __forceinline__ uint64_t lds64(const uint8_t* p) {
  return *reinterpret_cast<const uint64_t*>(p);
}

// Sum over one lane's words w = s + lane + 32 j (j < J) of a segment [s, e)
// that lies in one block: a += sum v, b += sum (w+1) v, with the (w+1)
// weights folded in once at the end from two running sums (T1 = sum v,
// T2 = sum_j sum_{i<j} v_i, so sum_j j v_j = (J-1) T1 - T2).  Interior words
// only (no masking); word w's bytes start at A0 + 8 (w - W0), shifted by sh.
__device__ __forceinline__ void segment_sums(const uint8_t* A0, int64_t W0, int sh, int64_t s,
                                             int64_t e, int lane, uint64_t& a, uint64_t& b) {
  const int64_t w0 = s + lane;
  if (w0 >= e) return;
  const uint64_t J = static_cast<uint64_t>((e - w0 + 31) / 32);
  const uint8_t* q = A0 + 8 * (w0 - W0);
  uint64_t t1 = 0, t2 = 0;
  if (sh == 0) {
#pragma unroll 4
    for (uint64_t j = 0; j < J; ++j, q += 256) {
      t2 += t1;
      t1 += lds64(q);
    }
  } else {
    const int rs = 8 * sh, ls = 64 - 8 * sh;
#pragma unroll 4
    for (uint64_t j = 0; j < J; ++j, q += 256) {
      t2 += t1;
      t1 += (lds64(q) >> rs) | (lds64(q + 8) << ls);
    }
  }
  a += t1;
  b += (static_cast<uint64_t>(w0) + 1) * t1 + 32 * ((J - 1) * t1 - t2);
}

__device__ void checksum_piece(const uint8_t* stage, const Piece& pc, int warp_c, int lane,
                               unsigned long long* block_sums, int word_shift) {
  const int r = static_cast<int>(reinterpret_cast<uintptr_t>(pc.src) & 15);
  const int64_t g0 = pc.glob;
  const int64_t W0 = g0 >> 3, W1 = (g0 + pc.bytes - 1) >> 3;
  const int64_t nw = W1 - W0 + 1;
  const int64_t q0 = W0 + nw * warp_c / kConsumerWarps;
  const int64_t q1 = W0 + nw * (warp_c + 1) / kConsumerWarps;
  if (q0 >= q1) return;  // uniform per warp
  // word W0's first byte sits at stage[p0], p0 = r + 8 W0 - g0 in [r-7, r];
  // the 8-byte-aligned loads below may touch up to 8 bytes of neighbouring
  // shared memory before the stage, only ever for masked-off bytes
  const int p0 = r + static_cast<int>(8 * W0 - g0);
  const int sh = p0 & 7;
  const uint8_t* A0 = stage + (p0 & ~7);
  const int64_t blkA = q0 >> word_shift;
  const int64_t WB = (blkA + 1) << word_shift;  // first word of the next block
  uint64_t a0 = 0, b0 = 0, a1 = 0, b1 = 0;
  // interior words (the piece's first and last words may be partial)
  const int64_t lo = max(q0, W0 + 1), hi = min(q1, W1);
  if (lo < hi) {
    segment_sums(A0, W0, sh, lo, min(hi, WB), lane, a0, b0);
    segment_sums(A0, W0, sh, max(lo, WB), hi, lane, a1, b1);
  }
  // the (possibly partial) first and last words, one lane each
  for (int end = 0; end < 2; ++end) {
    const int64_t w = end ? W1 : W0;
    if ((end && W1 == W0) || w < q0 || w >= q1 || lane != end) continue;
    const int k0 = static_cast<int>(8 * w - g0);
    const uint8_t* q = A0 + 8 * (w - W0);
    uint64_t v = sh ? (lds64(q) >> (8 * sh)) | (lds64(q + 8) << (64 - 8 * sh)) : lds64(q);
    const int lo_t = max(0, -k0), hi_t = min(8, pc.bytes - k0);
    const uint64_t keep = (hi_t >= 8 ? ~uint64_t{0} : ((uint64_t{1} << (8 * hi_t)) - 1)) &
                          ~((uint64_t{1} << (8 * lo_t)) - 1);
    v &= keep;
    const uint64_t wi = static_cast<uint64_t>(w) + 1;
    if (w < WB) {
      a0 += v;
      b0 += wi * v;
    } else {
      a1 += v;
      b1 += wi * v;
    }
  }
  const bool two = __any_sync(0xffffffffu, (a1 | b1) != 0);  // block boundary inside
  a0 = warp_sum64(a0);
  b0 = warp_sum64(b0);
  if (two) {
    a1 = warp_sum64(a1);
    b1 = warp_sum64(b1);
  }
  if (lane == 0) {
    if (a0 | b0) {
      atomicAdd(block_sums + 2 * blkA, static_cast<unsigned long long>(a0));
      atomicAdd(block_sums + 2 * blkA + 1, static_cast<unsigned long long>(b0));
    }
    if (a1 | b1) {
      atomicAdd(block_sums + 2 * (blkA + 1), static_cast<unsigned long long>(a1));
      atomicAdd(block_sums + 2 * (blkA + 1) + 1, static_cast<unsigned long long>(b1));
    }
  }
}

// The piece's vectors realigned by a compile-time byte offset OFF (1..15):
// four funnel shifts with constant word indices per 16-byte vector (the
// select chain of realign() costs ~60 instructions per vector; all-local
// programs — replica-aware recoveries, config D's 2->1 — are bound by it).
template <int OFF>
__device__ __forceinline__ void copy_realigned(uint8_t* db, const uint8_t* sb, int nv, int ctid) {
  constexpr int kC = 32 * kConsumerWarps;
  constexpr int ws = OFF >> 2, bs = (OFF & 3) * 8;
#pragma unroll 4
  for (int j = ctid; j < nv; j += kC) {
    const uint4 a = lds128(sb + 16 * j), b = lds128(sb + 16 * j + 16);
    const uint32_t x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint4 o;
    o.x = __funnelshift_r(x[ws + 0], x[ws + 1], bs);
    o.y = __funnelshift_r(x[ws + 1], x[ws + 2], bs);
    o.z = __funnelshift_r(x[ws + 2], x[ws + 3], bs);
    o.w = __funnelshift_r(x[ws + 3], x[ws + 4], bs);
    st_plain(db + 16 * j, o);
  }
}

// Consumers write one staged piece.  `stage` holds the source window that
// starts at floor16(pc.src); destination byte x lives at stage[x - dst + r].
__device__ __forceinline__ void write_piece(const uint8_t* stage, const Piece& pc, int ctid) {
  constexpr int kC = 32 * kConsumerWarps;
  const int r = static_cast<int>(reinterpret_cast<uintptr_t>(pc.src) & 15);
  const int head = min(pc.bytes, static_cast<int32_t>((16 - (reinterpret_cast<uintptr_t>(pc.dst) & 15)) & 15));
  const int nv = (pc.bytes - head) >> 4;
  const int tail = (pc.bytes - head) & 15;
  if (ctid < head) pc.dst[ctid] = stage[r + ctid];
  if (ctid >= 32 && ctid < 32 + tail) {
    const int k = head + 16 * nv + (ctid - 32);
    pc.dst[k] = stage[r + k];
  }
  uint8_t* db = pc.dst + head;
  const int off = (r + head) & 15;          // uniform per piece
  const uint8_t* sb = stage + ((r + head) & ~15);
  if (off == 0) {
#pragma unroll 4
    for (int j = ctid; j < nv; j += kC) st_plain(db + 16 * j, lds128(sb + 16 * j));
  } else {
    switch (off) {  // uniform per piece
      case 1: copy_realigned<1>(db, sb, nv, ctid); break;
      case 2: copy_realigned<2>(db, sb, nv, ctid); break;
      case 3: copy_realigned<3>(db, sb, nv, ctid); break;
      case 4: copy_realigned<4>(db, sb, nv, ctid); break;
      case 5: copy_realigned<5>(db, sb, nv, ctid); break;
      case 6: copy_realigned<6>(db, sb, nv, ctid); break;
      case 7: copy_realigned<7>(db, sb, nv, ctid); break;
      case 8: copy_realigned<8>(db, sb, nv, ctid); break;
      case 9: copy_realigned<9>(db, sb, nv, ctid); break;
      case 10: copy_realigned<10>(db, sb, nv, ctid); break;
      case 11: copy_realigned<11>(db, sb, nv, ctid); break;
      case 12: copy_realigned<12>(db, sb, nv, ctid); break;
      case 13: copy_realigned<13>(db, sb, nv, ctid); break;
      case 14: copy_realigned<14>(db, sb, nv, ctid); break;
      default: copy_realigned<15>(db, sb, nv, ctid); break;
    }
  }
}

__global__ void __launch_bounds__(kThreads, 2) staged_copy_kernel(const CopyItem* __restrict__ items,
                                                               int64_t n_remote,
                                                               int64_t remote_pieces,
                                                               int64_t n_local,
                                                               int64_t local_pieces,
                                                               int remote_ctas,
                                                               unsigned long long* block_sums,
                                                               int word_shift,
                                                               const int* abort_flag) {
  // gated launch: a failed barrier upstream in stream order vetoes the copy
  if (abort_flag != nullptr && *reinterpret_cast<const volatile int*>(abort_flag) != 0) return;
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ __align__(8) uint64_t empty[kStages];
  // the producer resolves each piece once (binary search over the items)
  // and hands it to the consumers with the stage: the mbarrier's
  // arrive (release) / wait (acquire) orders these plain shared stores
  __shared__ Piece staged[kStages];

  const bool remote = static_cast<int>(blockIdx.x) < remote_ctas;
  const CopyItem* list = remote ? items : items + n_remote;
  const int64_t n_items = remote ? n_remote : n_local;
  const int64_t n_pieces = remote ? remote_pieces : local_pieces;
  const int64_t first = remote ? blockIdx.x : blockIdx.x - remote_ctas;
  const int64_t step = remote ? remote_ctas : static_cast<int64_t>(gridDim.x) - remote_ctas;
  if (n_items == 0 || step <= 0 || first >= n_pieces) return;  // uniform per CTA
  const int64_t mine = (n_pieces - first + step - 1) / step;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {  // producer
    if (lane == 0) {
      ItemCursor cur;
      for (int64_t k = 0; k < mine; ++k) {
        const int s = static_cast<int>(k % kStages);
        if (k >= kStages) {
          mbar_wait(&empty[s], static_cast<uint32_t>(((k / kStages) - 1) & 1));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const int64_t p = first + k * step;
        const Piece pc = piece_at(cur.at(list, n_items, p), p);
        staged[s] = pc;
        const uintptr_t s0 = reinterpret_cast<uintptr_t>(pc.src) & ~uintptr_t{15};
        const uintptr_t s1 = (reinterpret_cast<uintptr_t>(pc.src) + pc.bytes + 15) & ~uintptr_t{15};
        const uint32_t n = static_cast<uint32_t>(s1 - s0);
        mbar_expect_tx(&full[s], n);
        tma_load(ring + s * kStageBytes, reinterpret_cast<const void*>(s0), n, &full[s]);
      }
    }
    return;
  }

  const int ctid = threadIdx.x - 32;  // consumer thread id
  for (int64_t k = 0; k < mine; ++k) {
    const int s = static_cast<int>(k % kStages);
    mbar_wait(&full[s], static_cast<uint32_t>((k / kStages) & 1));
    const Piece pc = staged[s];
    const uint8_t* stage = ring + s * kStageBytes;
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(pc.src) | reinterpret_cast<uintptr_t>(pc.dst)) & 15) == 0;
    const bool bulk = !pc.no_store && aligned && pc.bytes >= 16;
    if (pc.no_store) {
      // retained in place: only checksummed below, nothing to move
    } else if (bulk) {
      // 16-byte-congruent piece: one bulk shared->global store of the body
      // (no register traffic); the <16-byte tail by byte stores
      const int body = pc.bytes & ~15;
      if (ctid == 0) {
        tma_store(pc.dst, stage, static_cast<uint32_t>(body));
        bulk_commit();
      }
      if (ctid >= 32 && ctid < 32 + (pc.bytes - body)) pc.dst[body + ctid - 32] = stage[body + ctid - 32];
    } else {
      write_piece(stage, pc, ctid);
    }
    // verification on arrival, overlapped with the bulk store's smem read
    if (block_sums != nullptr && pc.glob >= 0)
      checksum_piece(stage, pc, warp - 1, lane, block_sums, word_shift);
    if (bulk && ctid == 0) bulk_wait_read<0>();  // the stage may be reused once read
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (ctid == 0) bulk_wait_all();  // bulk stores complete before the kernel retires
}

}  // namespace
}  // namespace ew

using namespace ew;

struct ew_copy_program {
  int device = -1;
  int64_t n_remote = 0, n_local = 0, remote_pieces = 0, local_pieces = 0;
  int64_t remote_bytes = 0, local_bytes = 0, copies = 0;
  CopyItem* d_items = nullptr;
  int word_shift = -1;  // verified programs: log2(block bytes / 8)
  int64_t n_blocks = 0;  // global blocks covered by the block sums
};

namespace {

int build_program(std::vector<CopyItem> remote, std::vector<CopyItem> local,
                  ew_copy_program** out) {
  auto* p = new ew_copy_program();
  int64_t base = 0;
  for (CopyItem& it : remote) {
    it.piece_base = base;
    base += pieces_of(it.dst, it.bytes);
    p->remote_bytes += it.bytes;
  }
  p->remote_pieces = base;
  base = 0;
  for (CopyItem& it : local) {
    it.piece_base = base;
    base += pieces_of(it.dst, it.bytes);
    p->local_bytes += it.bytes;
  }
  p->local_pieces = base;
  p->n_remote = static_cast<int64_t>(remote.size());
  p->n_local = static_cast<int64_t>(local.size());
  p->copies = p->n_remote + p->n_local;
  std::vector<CopyItem> all(remote);
  all.insert(all.end(), local.begin(), local.end());
  cudaError_t e = cudaGetDevice(&p->device);
  if (e == cudaSuccess && !all.empty()) {
    e = cudaMalloc(&p->d_items, all.size() * sizeof(CopyItem));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_items, all.data(), all.size() * sizeof(CopyItem),
                     cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(staged_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmem);
  if (e != cudaSuccess) {
    if (p->d_items) cudaFree(p->d_items);
    delete p;
    return cuda_status(e, "ew_copy_program_create");
  }
  *out = p;
  return EW_OK;
}

}  // namespace

extern "C" {

static int create_program(const ew_copy_desc* descs, int64_t n, void* const* buf_table,
                          int table_ranks, int exec_rank, const ew_shardmap* new_map,
                          ew_copy_program** out) {
  if (out == nullptr || (n > 0 && (descs == nullptr || buf_table == nullptr)) || table_ranks <= 0)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_copy_program_create: bad arguments");
  *out = nullptr;
  std::vector<CopyItem> remote, local;
  // Remote copies in ring order of their peer (exec+1, exec+2, ...): CTAs
  // sweep items in order, so the receivers of a pull (or the targets of a
  // push) start on different peers instead of all hitting the same one.
  std::vector<int64_t> order(static_cast<std::size_t>(std::max<int64_t>(n, 0)));
  for (int64_t i = 0; i < n; ++i) order[static_cast<std::size_t>(i)] = i;
  auto peer_of = [&](const ew_copy_desc& c) {
    const int p = (c.src_rank != exec_rank) ? c.src_rank : c.dst_rank;
    return (p - exec_rank + table_ranks) % table_ranks;
  };
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return peer_of(descs[a]) < peer_of(descs[b]);
  });
  constexpr int kNewRole = 2;  // b200::BufRole::New
  for (const int64_t i : order) {
    const ew_copy_desc& c = descs[i];
    if (c.bytes < 0 || c.src_role < 0 || c.src_role > 2 || c.dst_role < 0 || c.dst_role > 2 ||
        c.src_rank < 0 || c.src_rank >= table_ranks || c.dst_rank < 0 ||
        c.dst_rank >= table_ranks)
      return set_error(EW_ERR_INVALID_ARGUMENT,
                       "copy descriptor " + std::to_string(i) + " out of table range");
    if (c.bytes == 0) continue;
    const uint8_t* src =
        static_cast<const uint8_t*>(buf_table[c.src_role * table_ranks + c.src_rank]);
    uint8_t* dst = static_cast<uint8_t*>(buf_table[c.dst_role * table_ranks + c.dst_rank]);
    if (src == nullptr || dst == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT,
                       "copy descriptor " + std::to_string(i) + " refers to an unmapped buffer");
    // in-place reshards alias OLD and NEW: retained bytes already in place
    const bool in_place = src + c.src_off == dst + c.dst_off;
    // remote = the copy crosses NVLink (the other end is not exec_rank)
    const bool crosses = c.dst_rank != exec_rank || c.src_rank != exec_rank;
    const bool tracked = new_map != nullptr && c.dst_role == kNewRole && c.dst_rank == exec_rank;
    if (!tracked) {
      if (!in_place)
        (crosses ? remote : local).push_back({src + c.src_off, dst + c.dst_off, c.bytes, 0, -1, 0});
      continue;
    }
    // label the landed bytes with the global position their destination
    // offset has in NEW's segment map (independent of the plan's interval),
    // splitting at segment boundaries
    int64_t off = c.dst_off, left = c.bytes, soff = c.src_off;
    const auto& segs = new_map->h_segs;
    while (left > 0) {
      auto it = std::upper_bound(segs.begin(), segs.end(), off,
                                 [](int64_t v, const DevSeg& sg) { return v < sg.local_off; });
      if (it == segs.begin())
        return set_error(EW_ERR_COVERAGE_MISMATCH, "copy lands outside NEW's segment map");
      const DevSeg& sg = *(it - 1);
      if (off >= sg.local_off + sg.length)
        return set_error(EW_ERR_COVERAGE_MISMATCH, "copy lands outside NEW's segment map");
      const int64_t take = std::min(left, sg.local_off + sg.length - off);
      const int64_t glob = sg.global_lo + (off - sg.local_off);
      (crosses ? remote : local)
          .push_back({src + soff, dst + off, take, 0, glob, in_place ? 1 : 0});
      off += take;
      soff += take;
      left -= take;
    }
  }
  const int rc = build_program(std::move(remote), std::move(local), out);
  if (rc == EW_OK && new_map != nullptr) {
    (*out)->word_shift = new_map->block_shift - 3;
    const auto& segs = new_map->h_segs;
    (*out)->n_blocks = segs.empty() ? 0
        : ((segs.back().global_lo + segs.back().length - 1) >> new_map->block_shift) + 1;
  }
  return rc;
}

int ew_copy_program_create(const ew_copy_desc* descs, int64_t n, void* const* buf_table,
                           int table_ranks, int exec_rank, ew_copy_program** out) {
  return create_program(descs, n, buf_table, table_ranks, exec_rank, nullptr, out);
}

int ew_copy_program_create_verified(const ew_copy_desc* descs, int64_t n,
                                    void* const* buf_table, int table_ranks, int exec_rank,
                                    const ew_shardmap* new_map, ew_copy_program** out) {
  if (new_map == nullptr)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_copy_program_create_verified: NULL map");
  return create_program(descs, n, buf_table, table_ranks, exec_rank, new_map, out);
}

int ew_copy_program_create_raw(const void* const* srcs, void* const* dsts, const int64_t* bytes,
                               const int* is_remote, int64_t n, ew_copy_program** out) {
  if (out == nullptr || (n > 0 && (!srcs || !dsts || !bytes || !is_remote)))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_copy_program_create_raw: bad arguments");
  *out = nullptr;
  std::vector<CopyItem> remote, local;
  for (int64_t i = 0; i < n; ++i) {
    if (bytes[i] < 0) return set_error(EW_ERR_INVALID_ARGUMENT, "negative copy size");
    if (bytes[i] == 0) continue;
    CopyItem it{static_cast<const uint8_t*>(srcs[i]), static_cast<uint8_t*>(dsts[i]), bytes[i], 0,
                -1, 0};
    (is_remote[i] ? remote : local).push_back(it);
  }
  return build_program(std::move(remote), std::move(local), out);
}

void ew_copy_program_free(ew_copy_program* prog) {
  if (prog == nullptr) return;
  if (prog->d_items) cudaFree(prog->d_items);
  delete prog;
}

int ew_copy_program_stats(const ew_copy_program* prog, int64_t* n_copies, int64_t* remote_bytes,
                          int64_t* local_bytes) {
  if (prog == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL program");
  if (n_copies) *n_copies = prog->copies;
  if (remote_bytes) *remote_bytes = prog->remote_bytes;
  if (local_bytes) *local_bytes = prog->local_bytes;
  return EW_OK;
}

static int launch_program(const ew_copy_program* prog, int n_ctas, int remote_ctas,
                          uint64_t* block_sums, const int* abort_flag, ew_stream_t stream) {
  if (prog == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL program");
  if (prog->remote_pieces + prog->local_pieces == 0) return EW_OK;
  const int sms = num_sms();
  const bool mixed = prog->remote_pieces > 0 && prog->local_pieces > 0;
  // two 96 KiB rings per SM; a mixed program runs its local class one CTA
  // per SM: with the constant-shift realign the local copies would otherwise
  // finish early and press on the HBM the peers are still pulling from
  // (r01 A/B at 4->3: 148 local CTAs 10.95 ms vs 222 local CTAs 11.32 ms)
  // a local-only program (e.g. a replica-aware recovery whose sources are
  // all in this GPU's HBM) streams best with twice the resident CTAs: 15.72 GB
  // verified in 4.99 vs 5.28 ms (tools/local_copy_sweep.py)
  const bool local_only = prog->remote_pieces == 0;
  if (n_ctas <= 0) n_ctas = mixed ? sms + std::max(1, sms / 2) : local_only ? 4 * sms : 2 * sms;
  if (prog->remote_pieces == 0) remote_ctas = 0;
  else if (prog->local_pieces == 0) remote_ctas = n_ctas;
  else if (remote_ctas <= 0 || remote_ctas >= n_ctas)
    // NVLink class: half an SM's worth of CTAs per SM pair, verified or not
    // (N=4 sweep: 74 CTAs 11.07 ms verified vs 11.11 ms plain; 98 CTAs
    // 11.2 ms); callers sweep through the remote_ctas argument
    remote_ctas = std::max(1, std::min(n_ctas - 1, sms / 2));
  staged_copy_kernel<<<n_ctas, kThreads, kSmem, (cudaStream_t)stream>>>(
      prog->d_items, prog->n_remote, prog->remote_pieces, prog->n_local, prog->local_pieces,
      remote_ctas, reinterpret_cast<unsigned long long*>(block_sums), prog->word_shift,
      abort_flag);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

int ew_copy_program_launch(const ew_copy_program* prog, int n_ctas, int remote_ctas,
                           ew_stream_t stream) {
  return launch_program(prog, n_ctas, remote_ctas, nullptr, nullptr, stream);
}

int ew_copy_program_launch_guarded(const ew_copy_program* prog, int n_ctas, int remote_ctas,
                                   uint64_t* block_sums, const int* abort_flag,
                                   ew_stream_t stream) {
  if (prog != nullptr && block_sums != nullptr && prog->word_shift < 0)
    return set_error(EW_ERR_INVALID_ARGUMENT,
                     "ew_copy_program_launch_guarded: block sums need a verified program");
  return launch_program(prog, n_ctas, remote_ctas, prog && prog->word_shift >= 0 ? block_sums
                                                                                  : nullptr,
                        abort_flag, stream);
}

int ew_copy_program_launch_verified(const ew_copy_program* prog, int n_ctas, int remote_ctas,
                                    uint64_t* block_sums, ew_stream_t stream) {
  if (prog == nullptr || prog->word_shift < 0 || block_sums == nullptr)
    return set_error(EW_ERR_INVALID_ARGUMENT,
                     "ew_copy_program_launch_verified: needs a verified program and block sums");
  return launch_program(prog, n_ctas, remote_ctas, block_sums, nullptr, stream);
}

int ew_copy_program_num_blocks(const ew_copy_program* prog, int64_t* n_blocks) {
  if (prog == nullptr || n_blocks == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  *n_blocks = prog->n_blocks;
  return EW_OK;
}

}  // extern "C"
