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
//   consumers (4 warps): read the stage, realign it to the destination when
//     source and destination are not congruent mod 16 (byte-granular plans,
//     SURVEY fact 9), write 16-byte vectors, and byte-store the partial
//     vectors at copy ends so adjacent copies from other GPUs never race on a
//     vector; then release the stage on its "empty" mbarrier.
// Pieces are <= 16 KiB and cut at 16 KiB-aligned destination addresses, so
// no two pieces share a destination vector.
#include <algorithm>
#include <vector>

#include "ew_device.cuh"

namespace ew {
namespace {

constexpr int kConsumerWarps = 4;
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
};

__device__ __forceinline__ Piece piece_at(const CopyItem* list, int64_t n_items, int64_t p) {
  const CopyItem it = list[item_of_piece(list, n_items, p)];
  const uint64_t d = reinterpret_cast<uintptr_t>(it.dst);
  const uint64_t cut = (d / kPiece + static_cast<uint64_t>(p - it.piece_base)) * kPiece;
  const uint64_t lo = max(d, cut);
  const uint64_t hi = min(d + static_cast<uint64_t>(it.bytes), cut + kPiece);
  return Piece{it.src + (lo - d), it.dst + (lo - d), static_cast<int32_t>(hi - lo)};
}

__device__ __forceinline__ uint32_t pick(const uint32_t (&x)[8], int i) {
  uint32_t r = x[0];  // i is uniform per piece; the select chain stays in registers
#pragma unroll
  for (int k = 1; k < 8; ++k) r = (i == k) ? x[k] : r;
  return r;
}

// 16 bytes starting at byte `off` (1..15) of the 32-byte pair (a, b).
__device__ __forceinline__ uint4 realign(const uint4& a, const uint4& b, int off) {
  const uint32_t x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  const int ws = off >> 2;
  const int bs = (off & 3) * 8;
  uint4 o;
  o.x = __funnelshift_r(pick(x, ws + 0), pick(x, ws + 1), bs);
  o.y = __funnelshift_r(pick(x, ws + 1), pick(x, ws + 2), bs);
  o.z = __funnelshift_r(pick(x, ws + 2), pick(x, ws + 3), bs);
  o.w = __funnelshift_r(pick(x, ws + 3), pick(x, ws + 4), bs);
  return o;
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
#pragma unroll 4
    for (int j = ctid; j < nv; j += kC)
      st_plain(db + 16 * j, realign(lds128(sb + 16 * j), lds128(sb + 16 * j + 16), off));
  }
}

__global__ void __launch_bounds__(kThreads) staged_copy_kernel(const CopyItem* __restrict__ items,
                                                               int64_t n_remote,
                                                               int64_t remote_pieces,
                                                               int64_t n_local,
                                                               int64_t local_pieces,
                                                               int remote_ctas) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ __align__(8) uint64_t empty[kStages];

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
      for (int64_t k = 0; k < mine; ++k) {
        const int s = static_cast<int>(k % kStages);
        if (k >= kStages) {
          mbar_wait(&empty[s], static_cast<uint32_t>(((k / kStages) - 1) & 1));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const Piece pc = piece_at(list, n_items, first + k * step);
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
    const Piece pc = piece_at(list, n_items, first + k * step);
    const uint8_t* stage = ring + s * kStageBytes;
    const bool aligned =
        ((reinterpret_cast<uintptr_t>(pc.src) | reinterpret_cast<uintptr_t>(pc.dst)) & 15) == 0;
    if (aligned && pc.bytes >= 16) {
      // 16-byte-congruent piece: one bulk shared->global store of the body
      // (no register traffic); the <16-byte tail by byte stores
      const int body = pc.bytes & ~15;
      if (ctid == 0) {
        tma_store(pc.dst, stage, static_cast<uint32_t>(body));
        bulk_commit();
      }
      if (ctid >= 32 && ctid < 32 + (pc.bytes - body)) pc.dst[body + ctid - 32] = stage[body + ctid - 32];
      if (ctid == 0) bulk_wait_read<0>();  // the stage may be reused once read
    } else {
      write_piece(stage, pc, ctid);
    }
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

int ew_copy_program_create(const ew_copy_desc* descs, int64_t n, void* const* buf_table,
                           int table_ranks, int exec_rank, ew_copy_program** out) {
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
    if (src + c.src_off == dst + c.dst_off) continue;
    // remote = the copy crosses NVLink (the other end is not exec_rank)
    const bool crosses = c.dst_rank != exec_rank || c.src_rank != exec_rank;
    (crosses ? remote : local).push_back({src + c.src_off, dst + c.dst_off, c.bytes, 0});
  }
  return build_program(std::move(remote), std::move(local), out);
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
    CopyItem it{static_cast<const uint8_t*>(srcs[i]), static_cast<uint8_t*>(dsts[i]), bytes[i], 0};
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

int ew_copy_program_launch(const ew_copy_program* prog, int n_ctas, int remote_ctas,
                           ew_stream_t stream) {
  if (prog == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL program");
  if (prog->remote_pieces + prog->local_pieces == 0) return EW_OK;
  const int sms = num_sms();
  if (n_ctas <= 0) n_ctas = 2 * sms;  // two 96 KiB rings per SM
  if (prog->remote_pieces == 0) remote_ctas = 0;
  else if (prog->local_pieces == 0) remote_ctas = n_ctas;
  else if (remote_ctas <= 0 || remote_ctas >= n_ctas) remote_ctas = std::max(1, n_ctas / 4);
  staged_copy_kernel<<<n_ctas, kThreads, kSmem, (cudaStream_t)stream>>>(
      prog->d_items, prog->n_remote, prog->remote_pieces, prog->n_local, prog->local_pieces,
      remote_ctas);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

}  // extern "C"
