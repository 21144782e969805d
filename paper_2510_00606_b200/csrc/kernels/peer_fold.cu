// (d) Weighted reduce fused with its collective over NVLink peer memory.
//
// Same arithmetic as ew_weighted_fold + NCCL int64 all-reduce (each unit
// quantised once, q = rint(w*g*2^F), exact int64 sums -> bit-identical for
// every world size and split), but the collective is the kernel itself:
//   reduce-scatter: GPU r reads element chunk r of EVERY unit of every rank
//     straight from peer HBM (CUDA IPC mappings over NVSwitch), sums the
//     quantised terms in registers and writes its fp32 output chunk;
//   all-gather: GPU r pulls the other ranks' output chunks (staged-copy path).
// NVLink bytes per GPU: (N-1)/N * n * (4 B per unit + 4 B), versus 2 *
// (N-1)/N * n * 8 B for the int64 NCCL all-reduce, and no int64 accumulator
// array in HBM.  The communicator edit for a departed rank is dropping its
// pointers (no NCCL communicator to shrink).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "ew_device.cuh"

namespace ew {
namespace {

struct PeerUnit {
  const float* p;
  double w;
};

// TMA-staged reduce-scatter (up to kPfUnitsMax units): one producer lane
// bulk-loads the same 4 KiB slice of every unit — local or in peer HBM — into
// a shared-memory stage (one mbarrier per stage), four consumer warps
// quantise-and-sum the slices from shared memory and write the fp32 output
// chunk.  The loads keep ~kPfStages x U x 4 KiB in flight per CTA without
// register traffic, which is what NVLink latency needs.
constexpr int kPfUnitsMax = 8;

constexpr int kPfSlice = 4096;  // bytes per unit per stage = 256 float4
constexpr int kPfStages = 4;    // ring depth
constexpr int kPfStagesMax = 8;
constexpr int kPfCtasPerSm = 2;
constexpr int kPfConsumers = 4;
constexpr int kPfThreads = 32 * (kPfConsumers + 1);

// kI64: the units are per-rank int64 accumulators (32 B per group of 4
// elements instead of 16), summed without weights.
template <bool kI64>
__global__ void __launch_bounds__(kPfThreads) peer_fold_staged_kernel(
    const PeerUnit* __restrict__ units, int n_units, int64_t lo4, int64_t hi4, double scale,
    double inv_scale, float* __restrict__ out, int slice, int stages) {
  constexpr int kGroupBytes = kI64 ? 32 : 16;
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kPfStagesMax];
  __shared__ __align__(8) uint64_t empty[kPfStagesMax];
  const int64_t per_piece = slice / kGroupBytes;
  const int64_t n_pieces = (hi4 - lo4 + per_piece - 1) / per_piece;
  const int64_t first = blockIdx.x, step = gridDim.x;
  if (first >= n_pieces) return;
  const int64_t mine = (n_pieces - first + step - 1) / step;
  const int stage_bytes = n_units * slice;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPfConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane != 0) return;
    for (int64_t k = 0; k < mine; ++k) {
      const int s = static_cast<int>(k % stages);
      if (k >= stages) {
        mbar_wait(&empty[s], static_cast<uint32_t>(((k / stages) - 1) & 1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      const int64_t start = lo4 + (first + k * step) * per_piece;
      const uint32_t bytes = static_cast<uint32_t>(kGroupBytes * min(per_piece, hi4 - start));
      mbar_expect_tx(&full[s], bytes * n_units);
      for (int u = 0; u < n_units; ++u)
        tma_load(ring + s * stage_bytes + u * slice,
                 reinterpret_cast<const uint8_t*>(units[u].p) + kGroupBytes * start, bytes,
                 &full[s]);
    }
    return;
  }
  double w[kPfUnitsMax];
#pragma unroll
  for (int u = 0; u < kPfUnitsMax; ++u) w[u] = u < n_units ? units[u].w : 0.0;
  const int ctid = threadIdx.x - 32;
  for (int64_t k = 0; k < mine; ++k) {
    const int s = static_cast<int>(k % stages);
    mbar_wait(&full[s], static_cast<uint32_t>((k / stages) & 1));
    const int64_t start = lo4 + (first + k * step) * per_piece;
    const int nf4 = static_cast<int>(min(per_piece, hi4 - start));
    const uint8_t* stage = ring + s * stage_bytes;
    for (int j = ctid; j < nf4; j += 32 * kPfConsumers) {
      long long a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
      for (int u = 0; u < kPfUnitsMax; ++u) {
        if (u < n_units) {
          if (kI64) {  // wrapping int64 adds, like ncclInt64
            const uint4 x = lds128(stage + u * slice + 32 * j);
            const uint4 y = lds128(stage + u * slice + 32 * j + 16);
            a0 = static_cast<long long>(static_cast<unsigned long long>(a0) +
                                        (static_cast<unsigned long long>(x.y) << 32 | x.x));
            a1 = static_cast<long long>(static_cast<unsigned long long>(a1) +
                                        (static_cast<unsigned long long>(x.w) << 32 | x.z));
            a2 = static_cast<long long>(static_cast<unsigned long long>(a2) +
                                        (static_cast<unsigned long long>(y.y) << 32 | y.x));
            a3 = static_cast<long long>(static_cast<unsigned long long>(a3) +
                                        (static_cast<unsigned long long>(y.w) << 32 | y.z));
          } else {
            const uint4 raw = lds128(stage + u * slice + 16 * j);
            a0 += __double2ll_rn((w[u] * static_cast<double>(__uint_as_float(raw.x))) * scale);
            a1 += __double2ll_rn((w[u] * static_cast<double>(__uint_as_float(raw.y))) * scale);
            a2 += __double2ll_rn((w[u] * static_cast<double>(__uint_as_float(raw.z))) * scale);
            a3 += __double2ll_rn((w[u] * static_cast<double>(__uint_as_float(raw.w))) * scale);
          }
        }
      }
      reinterpret_cast<float4*>(out)[start + j] =
          make_float4(static_cast<float>(static_cast<double>(a0) * inv_scale),
                      static_cast<float>(static_cast<double>(a1) * inv_scale),
                      static_cast<float>(static_cast<double>(a2) * inv_scale),
                      static_cast<float>(static_cast<double>(a3) * inv_scale));
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// Rank `rank`'s chunk of float4 groups: [lo4, hi4); the last rank also owns
// the scalar tail [4*n4, n).
__global__ void __launch_bounds__(256) peer_fold_kernel(const PeerUnit* __restrict__ units,
                                                        int n_units, int64_t lo4, int64_t hi4,
                                                        int64_t tail_lo, int64_t n, double scale,
                                                        double inv_scale, float* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  constexpr int kDepth = 2;
  for (int64_t i0 = lo4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < hi4;
       i0 += kDepth * stride) {
    long long s[kDepth][4] = {};
    for (int k = 0; k < n_units; ++k) {
      const float4* src = reinterpret_cast<const float4*>(units[k].p);
      const double w = units[k].w;
      float4 g[kDepth];
#pragma unroll
      for (int d = 0; d < kDepth; ++d) {
        const int64_t i = i0 + d * stride;
        g[d] = i < hi4 ? src[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int d = 0; d < kDepth; ++d) {
        s[d][0] += __double2ll_rn((w * static_cast<double>(g[d].x)) * scale);
        s[d][1] += __double2ll_rn((w * static_cast<double>(g[d].y)) * scale);
        s[d][2] += __double2ll_rn((w * static_cast<double>(g[d].z)) * scale);
        s[d][3] += __double2ll_rn((w * static_cast<double>(g[d].w)) * scale);
      }
    }
#pragma unroll
    for (int d = 0; d < kDepth; ++d) {
      const int64_t i = i0 + d * stride;
      if (i >= hi4) break;
      reinterpret_cast<float4*>(out)[i] =
          make_float4(static_cast<float>(static_cast<double>(s[d][0]) * inv_scale),
                      static_cast<float>(static_cast<double>(s[d][1]) * inv_scale),
                      static_cast<float>(static_cast<double>(s[d][2]) * inv_scale),
                      static_cast<float>(static_cast<double>(s[d][3]) * inv_scale));
    }
  }
  for (int64_t i = tail_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    long long acc = 0;
    for (int k = 0; k < n_units; ++k)
      acc += __double2ll_rn((units[k].w * static_cast<double>(units[k].p[i])) * scale);
    out[i] = static_cast<float>(static_cast<double>(acc) * inv_scale);
  }
}

// Reduce-scatter of per-rank int64 accumulators (each rank already folded
// its micro-batch units locally, accumulate=1): GPU r sums element chunk r of
// every rank's accumulator straight from peer HBM (wrapping int64 adds, like
// ncclInt64), dequantises and writes its fp32 chunk.  8 B/element cross
// NVLink per peer instead of the 2 x 8 B of an int64 all-reduce.
__global__ void __launch_bounds__(256) peer_sum_i64_kernel(const PeerUnit* __restrict__ accs,
                                                           int n_accs, int64_t lo4, int64_t hi4,
                                                           int64_t tail_lo, int64_t n,
                                                           double inv_scale,
                                                           float* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  constexpr int kDepth = 2;
  for (int64_t i0 = lo4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < hi4;
       i0 += kDepth * stride) {
    unsigned long long sum[kDepth][4] = {};
    for (int k = 0; k < n_accs; ++k) {
      const longlong2* src = reinterpret_cast<const longlong2*>(accs[k].p);
      longlong2 x[kDepth][2];
#pragma unroll
      for (int d = 0; d < kDepth; ++d) {
        const int64_t i = i0 + d * stride;
        if (i < hi4) {
          x[d][0] = src[2 * i];
          x[d][1] = src[2 * i + 1];
        } else {
          x[d][0] = x[d][1] = make_longlong2(0, 0);
        }
      }
#pragma unroll
      for (int d = 0; d < kDepth; ++d) {
        sum[d][0] += static_cast<unsigned long long>(x[d][0].x);
        sum[d][1] += static_cast<unsigned long long>(x[d][0].y);
        sum[d][2] += static_cast<unsigned long long>(x[d][1].x);
        sum[d][3] += static_cast<unsigned long long>(x[d][1].y);
      }
    }
#pragma unroll
    for (int d = 0; d < kDepth; ++d) {
      const int64_t i = i0 + d * stride;
      if (i >= hi4) break;
      reinterpret_cast<float4*>(out)[i] = make_float4(
          static_cast<float>(static_cast<double>(static_cast<long long>(sum[d][0])) * inv_scale),
          static_cast<float>(static_cast<double>(static_cast<long long>(sum[d][1])) * inv_scale),
          static_cast<float>(static_cast<double>(static_cast<long long>(sum[d][2])) * inv_scale),
          static_cast<float>(static_cast<double>(static_cast<long long>(sum[d][3])) * inv_scale));
    }
  }
  for (int64_t i = tail_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    unsigned long long a = 0;
    for (int k = 0; k < n_accs; ++k)
      a += static_cast<unsigned long long>(reinterpret_cast<const long long*>(accs[k].p)[i]);
    out[i] = static_cast<float>(static_cast<double>(static_cast<long long>(a)) * inv_scale);
  }
}

// Device-side barrier across GPUs over peer memory: thread p stores `epoch`
// into slot [rank] of rank p's flag array (system-scope release), then waits
// until slot [p] of this rank's array reaches `epoch` (system-scope acquire).
// A bounded spin: after ~timeout_cycles the wait gives up and raises *err, so
// a missing peer surfaces as an error instead of a hung GPU.
__global__ void peer_barrier_kernel(unsigned long long* const* __restrict__ flags, int rank,
                                    int world, unsigned long long epoch, long long timeout_cycles,
                                    int* __restrict__ err) {
  const int p = threadIdx.x;
  if (p >= world) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flags[p] + rank), "l"(epoch)
               : "memory");
  const unsigned long long* mine = flags[rank] + p;
  const long long start = clock64();
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
    if (v >= epoch) break;
    if (clock64() - start > timeout_cycles) {
      atomicExch(err, 1);
      break;
    }
    __nanosleep(200);
  }
}

}  // namespace
}  // namespace ew

using namespace ew;

struct ew_peer_barrier {
  int world = 0, rank = 0;
  unsigned long long epoch = 0;
  unsigned long long** d_flags = nullptr;
  int* d_err = nullptr;
};

extern "C" {

int ew_peer_barrier_create(int world, int rank, unsigned long long* const* flag_ptrs,
                           ew_peer_barrier** out) {
  if (out == nullptr || world < 1 || world > 1024 || rank < 0 || rank >= world || !flag_ptrs)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_peer_barrier_create: bad arguments");
  for (int r = 0; r < world; ++r)
    if (flag_ptrs[r] == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL flag array");
  auto* b = new ew_peer_barrier();
  b->world = world;
  b->rank = rank;
  cudaError_t e = cudaMalloc(&b->d_flags, world * sizeof(unsigned long long*));
  if (e == cudaSuccess)
    e = cudaMemcpy(b->d_flags, flag_ptrs, world * sizeof(unsigned long long*), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&b->d_err, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(b->d_err, 0, sizeof(int));
  if (e != cudaSuccess) {
    if (b->d_flags) cudaFree(b->d_flags);
    if (b->d_err) cudaFree(b->d_err);
    delete b;
    return cuda_status(e, "ew_peer_barrier_create");
  }
  *out = b;
  return EW_OK;
}

int ew_peer_barrier_wait(ew_peer_barrier* b, double timeout_s, ew_stream_t stream) {
  if (b == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL barrier");
  ++b->epoch;
  const long long cycles = static_cast<long long>(timeout_s * 2.0e9);  // <= 2 GHz SM clock
  peer_barrier_kernel<<<1, 32 * ((b->world + 31) / 32), 0, (cudaStream_t)stream>>>(
      b->d_flags, b->rank, b->world, b->epoch, cycles, b->d_err);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

int ew_peer_barrier_timed_out(ew_peer_barrier* b, int* timed_out) {
  if (b == nullptr || timed_out == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  EW_CUDA_TRY(cudaMemcpy(timed_out, b->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  return EW_OK;
}

int ew_peer_barrier_error_flag(ew_peer_barrier* b, const int** flag) {
  if (b == nullptr || flag == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  *flag = b->d_err;
  return EW_OK;
}

void ew_peer_barrier_free(ew_peer_barrier* b) {
  if (b == nullptr) return;
  if (b->d_flags) cudaFree(b->d_flags);
  if (b->d_err) cudaFree(b->d_err);
  delete b;
}

}  // extern "C"

struct ew_peer_fold {
  int world = 0, rank = 0, n_units = 0;
  bool i64 = false;  // units are per-rank int64 accumulators (create_i64)
  int64_t n = 0, lo4 = 0, hi4 = 0, tail_lo = 0, tail_hi = 0;
  PeerUnit* d_units = nullptr;
  float* out = nullptr;
  ew_copy_program* gather = nullptr;
};

extern "C" {

static int peer_fold_create(int world, int rank, int64_t n_elems, const float* const* unit_ptrs,
                            const double* unit_weights, int n_units, float* const* out_ptrs,
                            bool i64, ew_peer_fold** out) {
  if (out == nullptr || world < 1 || rank < 0 || rank >= world || n_elems < 0 || n_units < 0 ||
      (n_units > 0 && (!unit_ptrs || !unit_weights)) || out_ptrs == nullptr)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_peer_fold_create: bad arguments");
  *out = nullptr;
  for (int k = 0; k < n_units; ++k)
    if (unit_ptrs[k] == nullptr || (reinterpret_cast<uintptr_t>(unit_ptrs[k]) & 15))
      return set_error(EW_ERR_INVALID_ARGUMENT, "unit pointers must be non-null and 16-byte aligned");
  for (int r = 0; r < world; ++r)
    if (out_ptrs[r] == nullptr || (reinterpret_cast<uintptr_t>(out_ptrs[r]) & 15))
      return set_error(EW_ERR_INVALID_ARGUMENT, "output pointers must be non-null and 16-byte aligned");
  auto* f = new ew_peer_fold();
  f->i64 = i64;
  f->world = world;
  f->rank = rank;
  f->n = n_elems;
  f->n_units = n_units;
  f->out = out_ptrs[rank];
  const int64_t n4 = n_elems / 4;
  auto lo_of = [&](int r) { return n4 * r / world; };
  f->lo4 = lo_of(rank);
  f->hi4 = lo_of(rank + 1);
  f->tail_lo = (rank == world - 1) ? 4 * n4 : n_elems;  // last rank owns the scalar tail
  std::vector<PeerUnit> units(static_cast<std::size_t>(n_units));
  for (int k = 0; k < n_units; ++k) units[k] = PeerUnit{unit_ptrs[k], unit_weights[k]};
  cudaError_t e = cudaSuccess;
  if (n_units > 0) {
    e = cudaMalloc(&f->d_units, units.size() * sizeof(PeerUnit));
    if (e == cudaSuccess)
      e = cudaMemcpy(f->d_units, units.data(), units.size() * sizeof(PeerUnit),
                     cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    if (f->d_units) cudaFree(f->d_units);
    delete f;
    return cuda_status(e, "ew_peer_fold_create");
  }
  // all-gather program: pull every other rank's chunk from its output buffer
  std::vector<const void*> srcs;
  std::vector<void*> dsts;
  std::vector<int64_t> bytes;
  std::vector<int> remote;
  // ring order (rank+1, rank+2, ...): CTAs work through the items in order,
  // so at any moment each peer's chunk is being read by one puller
  for (int step = 1; step < world; ++step) {
    const int r = (rank + step) % world;
    const int64_t lo = 4 * lo_of(r);
    const int64_t hi = (r == world - 1) ? n_elems : 4 * lo_of(r + 1);
    if (hi <= lo) continue;
    srcs.push_back(out_ptrs[r] + lo);
    dsts.push_back(out_ptrs[rank] + lo);
    bytes.push_back((hi - lo) * 4);
    remote.push_back(1);
  }
  if (!bytes.empty()) {
    if (int st = ew_copy_program_create_raw(srcs.data(), dsts.data(), bytes.data(), remote.data(),
                                            static_cast<int64_t>(bytes.size()), &f->gather)) {
      if (f->d_units) cudaFree(f->d_units);
      delete f;
      return st;
    }
  }
  *out = f;
  return EW_OK;
}

int ew_peer_fold_create(int world, int rank, int64_t n_elems, const float* const* unit_ptrs,
                        const double* unit_weights, int n_units, float* const* out_ptrs,
                        ew_peer_fold** out) {
  return peer_fold_create(world, rank, n_elems, unit_ptrs, unit_weights, n_units, out_ptrs,
                          false, out);
}

int ew_peer_fold_create_i64(int world, int rank, int64_t n_elems, const int64_t* const* acc_ptrs,
                            float* const* out_ptrs, ew_peer_fold** out) {
  if (acc_ptrs == nullptr || world < 1)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_peer_fold_create_i64: bad arguments");
  std::vector<const float*> p(static_cast<std::size_t>(world));
  std::vector<double> w(static_cast<std::size_t>(world), 0.0);
  for (int r = 0; r < world; ++r) p[r] = reinterpret_cast<const float*>(acc_ptrs[r]);
  return peer_fold_create(world, rank, n_elems, p.data(), w.data(), world, out_ptrs, true, out);
}

int ew_peer_fold_reduce_scatter(ew_peer_fold* f, int frac_bits, ew_stream_t stream) {
  if (f == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL peer fold");
  if (frac_bits > 1000 || frac_bits < -1000)
    return set_error(EW_ERR_INVALID_ARGUMENT, "frac_bits out of range");
  const int64_t work = std::max<int64_t>(f->hi4 - f->lo4, f->n - f->tail_lo);
  if (work <= 0) return EW_OK;
  if (f->n_units == 0) {
    EW_CUDA_TRY(cudaMemsetAsync(f->out + 4 * f->lo4, 0, (f->hi4 - f->lo4) * 16, (cudaStream_t)stream));
    if (f->n > f->tail_lo)
      EW_CUDA_TRY(cudaMemsetAsync(f->out + f->tail_lo, 0, (f->n - f->tail_lo) * 4, (cudaStream_t)stream));
    return EW_OK;
  }
  const double scale = std::ldexp(1.0, frac_bits), inv = std::ldexp(1.0, -frac_bits);
  if (f->i64 && (f->n_units > kPfUnitsMax || f->hi4 <= f->lo4)) {  // LDG fallback
    const int64_t work = std::max<int64_t>(f->hi4 - f->lo4, f->n - f->tail_lo);
    const int grid = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 8 * num_sms())));
    peer_sum_i64_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        f->d_units, f->n_units, f->lo4, f->hi4, f->tail_lo, f->n, inv, f->out);
    EW_CUDA_TRY(cudaGetLastError());
    return EW_OK;
  }
  if (f->n_units <= kPfUnitsMax && f->hi4 > f->lo4) {
    const int slice = kPfSlice;
    const int stages = kPfStages;
    const int smem = stages * f->n_units * slice;
    const auto kern = f->i64 ? peer_fold_staged_kernel<true> : peer_fold_staged_kernel<false>;
    EW_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int gb = f->i64 ? 32 : 16;
    const int64_t pieces = (f->hi4 - f->lo4 + slice / gb - 1) / (slice / gb);
    const int grid = static_cast<int>(
        std::min<int64_t>(pieces, kPfCtasPerSm * num_sms()));
    kern<<<grid, kPfThreads, smem, (cudaStream_t)stream>>>(
        f->d_units, f->n_units, f->lo4, f->hi4, scale, inv, f->out, slice, stages);
    EW_CUDA_TRY(cudaGetLastError());
    if (f->n > f->tail_lo) {  // scalar tail (last rank only)
      if (f->i64)
        peer_sum_i64_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(
            f->d_units, f->n_units, 0, 0, f->tail_lo, f->n, inv, f->out);
      else
        peer_fold_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(
            f->d_units, f->n_units, 0, 0, f->tail_lo, f->n, scale, inv, f->out);
      EW_CUDA_TRY(cudaGetLastError());
    }
    return EW_OK;
  }
  const int grid = static_cast<int>(std::min<int64_t>((work + 255) / 256, 8 * num_sms()));
  peer_fold_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      f->d_units, f->n_units, f->lo4, f->hi4, f->tail_lo, f->n, scale, inv, f->out);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

int ew_peer_fold_all_gather(ew_peer_fold* f, ew_stream_t stream) {
  if (f == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL peer fold");
  if (f->gather == nullptr) return EW_OK;
  return ew_copy_program_launch(f->gather, 0, 0, stream);
}

void ew_peer_fold_free(ew_peer_fold* f) {
  if (f == nullptr) return;
  if (f->d_units) cudaFree(f->d_units);
  if (f->gather) ew_copy_program_free(f->gather);
  delete f;
}

}  // extern "C"
