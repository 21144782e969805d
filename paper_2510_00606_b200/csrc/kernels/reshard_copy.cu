// (b) Reshard executor: the planner's TransferPlan lowered to copies and run
// as one kernel over NVLink/NVSwitch peer pointers plus local HBM.
//
// The reference only *times* a remap (remap_time, sim.cpp:452-483: max lane
// bytes / 25 GB/s).  Here each GPU runs one launch over its copy program
// (b200.hpp reshard_copies): the first CTAs stream the remote copies (push:
// 128-bit stores into IPC-mapped peer buffers), the remaining CTAs do the
// local ones (retained bytes that change packed position, ring-holder
// self-lanes).  Copies are byte-granular and src/dst may be mutually
// misaligned: destination vectors are always 16-byte aligned
// stores; a misaligned source is realigned in registers from two aligned
// 16-byte loads (neighbour lane's vector via warp shuffle); head/tail bytes
// use byte stores so adjacent copies from other GPUs never race on a vector.
// Work is cut into 64 KiB destination-aligned chunks (no two chunks share a
// 16-byte destination vector).
#include <algorithm>
#include <vector>

#include "ew_device.cuh"

namespace ew {
namespace {

constexpr int kThreads = 256;
constexpr int64_t kChunk = 64 * 1024;

struct CopyItem {
  const uint8_t* src;
  uint8_t* dst;
  int64_t bytes;
  int64_t chunk_base;  // first chunk id of this item within its class
};

__host__ __device__ __forceinline__ int64_t chunks_of(const uint8_t* dst, int64_t bytes) {
  if (bytes <= 0) return 0;
  const uint64_t d = reinterpret_cast<uintptr_t>(dst);
  return static_cast<int64_t>((d + bytes - 1) / kChunk - d / kChunk + 1);
}

__device__ __forceinline__ int64_t item_of_chunk(const CopyItem* items, int64_t n, int64_t c) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (items[mid].chunk_base <= c) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t pick(const uint32_t (&x)[8], int i) {
  // i is warp-uniform; unrolled select keeps x in registers
  uint32_t r = x[0];
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

// CTA-cooperative copy of n bytes src -> dst (any alignment).
__device__ __forceinline__ void copy_range(const uint8_t* __restrict__ s, uint8_t* __restrict__ d,
                                           int64_t n) {
  const int tid = threadIdx.x;
  const int64_t head = min(n, static_cast<int64_t>((16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15));
  const int64_t nv = (n - head) >> 4;
  const int64_t tail = (n - head) & 15;
  if (tid < head) d[tid] = s[tid];
  if (tid >= 32 && tid < 32 + tail) {
    const int64_t k = head + 16 * nv + (tid - 32);
    d[k] = s[k];
  }
  if (nv == 0) return;
  const uint8_t* sb = s + head;
  uint8_t* db = d + head;
  const int off = static_cast<int>(reinterpret_cast<uintptr_t>(sb) & 15);

  if (off == 0) {
    constexpr int U = 4;
    for (int64_t j0 = tid; j0 < nv; j0 += kThreads * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = j0 + u * kThreads;
        if (j < nv) v[u] = ld_stream(sb + 16 * j);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = j0 + u * kThreads;
        if (j < nv) st_plain(db + 16 * j, v[u]);
      }
    }
    return;
  }

  // misaligned source: lane l of a warp handles destination vector 32*g + l
  const uint8_t* sa = sb - off;  // aligned
  const int lane = tid & 31;
  const int warp = tid >> 5;
  constexpr int kWarps = kThreads / 32;
  const int64_t groups = (nv + 31) >> 5;
  for (int64_t g = warp; g < groups; g += kWarps) {
    const int64_t j = 32 * g + lane;
    uint4 a = make_uint4(0, 0, 0, 0), b = make_uint4(0, 0, 0, 0);
    if (j <= nv) a = ld_stream(sa + 16 * j);
    if (lane == 31 && j + 1 <= nv) b = ld_stream(sa + 16 * (j + 1));
    uint4 nb;
    nb.x = __shfl_down_sync(0xffffffffu, a.x, 1);
    nb.y = __shfl_down_sync(0xffffffffu, a.y, 1);
    nb.z = __shfl_down_sync(0xffffffffu, a.z, 1);
    nb.w = __shfl_down_sync(0xffffffffu, a.w, 1);
    if (lane != 31) b = nb;
    if (j < nv) st_plain(db + 16 * j, realign(a, b, off));
  }
}

__global__ void __launch_bounds__(kThreads) copy_kernel(const CopyItem* __restrict__ items,
                                                        int64_t n_remote, int64_t remote_chunks,
                                                        int64_t n_local, int64_t local_chunks,
                                                        int remote_ctas) {
  const bool remote = static_cast<int>(blockIdx.x) < remote_ctas;
  const CopyItem* list = remote ? items : items + n_remote;
  const int64_t n_items = remote ? n_remote : n_local;
  const int64_t n_chunks = remote ? remote_chunks : local_chunks;
  const int64_t first = remote ? blockIdx.x : blockIdx.x - remote_ctas;
  const int64_t step = remote ? remote_ctas : static_cast<int64_t>(gridDim.x) - remote_ctas;
  if (n_items == 0 || step <= 0) return;
  for (int64_t c = first; c < n_chunks; c += step) {
    const CopyItem it = list[item_of_chunk(list, n_items, c)];
    const uint64_t d = reinterpret_cast<uintptr_t>(it.dst);
    const uint64_t cb = (d / kChunk + (c - it.chunk_base)) * kChunk;
    const uint64_t lo = max(d, cb);
    const uint64_t hi = min(d + static_cast<uint64_t>(it.bytes), cb + kChunk);
    copy_range(it.src + (lo - d), it.dst + (lo - d), static_cast<int64_t>(hi - lo));
  }
}

}  // namespace
}  // namespace ew

using namespace ew;

struct ew_copy_program {
  int device = -1;
  int64_t n_remote = 0, n_local = 0;
  int64_t remote_chunks = 0, local_chunks = 0;
  int64_t remote_bytes = 0, local_bytes = 0;
  CopyItem* d_items = nullptr;
};

namespace {

int build_program(std::vector<CopyItem> remote, std::vector<CopyItem> local,
                  ew_copy_program** out) {
  auto* p = new ew_copy_program();
  int64_t base = 0;
  for (CopyItem& it : remote) {
    it.chunk_base = base;
    base += chunks_of(it.dst, it.bytes);
    p->remote_bytes += it.bytes;
  }
  p->remote_chunks = base;
  base = 0;
  for (CopyItem& it : local) {
    it.chunk_base = base;
    base += chunks_of(it.dst, it.bytes);
    p->local_bytes += it.bytes;
  }
  p->local_chunks = base;
  p->n_remote = static_cast<int64_t>(remote.size());
  p->n_local = static_cast<int64_t>(local.size());
  std::vector<CopyItem> all(remote);
  all.insert(all.end(), local.begin(), local.end());
  cudaError_t e = cudaGetDevice(&p->device);
  if (e == cudaSuccess && !all.empty()) {
    e = cudaMalloc(&p->d_items, all.size() * sizeof(CopyItem));
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_items, all.data(), all.size() * sizeof(CopyItem),
                     cudaMemcpyHostToDevice);
  }
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
  for (int64_t i = 0; i < n; ++i) {
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
    CopyItem it{src + c.src_off, dst + c.dst_off, c.bytes, 0};
    (c.dst_rank != exec_rank ? remote : local).push_back(it);
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
  if (n_copies) *n_copies = prog->n_remote + prog->n_local;
  if (remote_bytes) *remote_bytes = prog->remote_bytes;
  if (local_bytes) *local_bytes = prog->local_bytes;
  return EW_OK;
}

int ew_copy_program_launch(const ew_copy_program* prog, int n_ctas, int remote_ctas,
                           ew_stream_t stream) {
  if (prog == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL program");
  if (prog->remote_chunks + prog->local_chunks == 0) return EW_OK;
  const int sms = num_sms();
  if (n_ctas <= 0) n_ctas = 4 * sms;
  if (prog->remote_chunks == 0) remote_ctas = 0;
  else if (prog->local_chunks == 0) remote_ctas = n_ctas;
  else if (remote_ctas <= 0) {
    // NVLink-bound remote stream vs HBM-bound local stream (2 bytes of HBM
    // traffic per local byte): give each class CTAs in proportion to its time
    const double t_remote = static_cast<double>(prog->remote_bytes) / 750.0;
    const double t_local = 2.0 * static_cast<double>(prog->local_bytes) / 6000.0;
    remote_ctas = static_cast<int>(n_ctas * t_remote / (t_remote + t_local) + 0.5);
    remote_ctas = std::max(sms / 2, std::min(remote_ctas, n_ctas - sms / 2));
  }
  remote_ctas = std::max(0, std::min(remote_ctas, n_ctas));
  if (remote_ctas == n_ctas && prog->local_chunks > 0) n_ctas += sms;
  if (remote_ctas == 0 && prog->remote_chunks > 0) remote_ctas = std::min(n_ctas, sms);
  copy_kernel<<<n_ctas, kThreads, 0, (cudaStream_t)stream>>>(
      prog->d_items, prog->n_remote, prog->remote_chunks, prog->n_local, prog->local_chunks,
      remote_ctas);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

}  // extern "C"
