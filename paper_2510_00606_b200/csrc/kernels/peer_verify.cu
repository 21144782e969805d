// Reshard verification by checksum conservation, reduce-scattered over peer
// memory (recovery.hpp BlockVerifier).
//
// Each survivor r holds block-sum arrays (u64 [2 * n_blocks], kernel (a)'s
// spec): what its verified copy landed, and what its OLD shard / ring replica
// held before the change (from the per-step snapshot rows).  The move is
// correct (up to the checksum's linear collisions, ew_api.h) iff for every
// block word i
//     sum_{plus} a[i] == sum_{minus} b[i]   (mod 2^64).
// A survivor checks words [lo, hi) — its slice — reading every peer's arrays
// through IPC pointers over NVLink, and counts mismatching words: 16 B per
// array per word pair, ~23 MB per array at config B, spread over all GPUs.
#include <algorithm>
#include <vector>

#include "ew_device.cuh"

struct ew_block_verifier {
  const uint64_t** d_ptrs = nullptr;  // plus pointers then minus pointers
  int n_plus = 0, n_minus = 0;
  int64_t lo = 0, hi = 0;
};

namespace ew {
namespace {

__global__ void __launch_bounds__(256) conservation_kernel(const uint64_t* const* __restrict__ ptrs,
                                                           int n_plus, int n_minus, int64_t lo,
                                                           int64_t hi, unsigned* __restrict__ bad) {
  const int64_t n2 = (hi - lo) / 2;  // word pairs (s0, s1) of one block
  unsigned mine = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = lo + 2 * i;
    uint64_t d0 = 0, d1 = 0;
    for (int k = 0; k < n_plus; ++k) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(ptrs[k] + w);
      d0 += v.x;
      d1 += v.y;
    }
    for (int k = 0; k < n_minus; ++k) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(ptrs[n_plus + k] + w);
      d0 -= v.x;
      d1 -= v.y;
    }
    mine += (d0 != 0) + (d1 != 0);
  }
  mine = __reduce_add_sync(0xffffffffu, mine);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(bad, mine);
}

}  // namespace
}  // namespace ew

using namespace ew;

extern "C" {

int ew_block_verifier_create(const uint64_t* const* plus, int n_plus, const uint64_t* const* minus,
                             int n_minus, int64_t lo, int64_t hi, ew_block_verifier** out) {
  if (out == nullptr || n_plus < 0 || n_minus < 0 || n_plus + n_minus > 4096 || lo < 0 ||
      hi < lo || (lo & 1) || (hi & 1) || (n_plus && !plus) || (n_minus && !minus))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_block_verifier_create: bad arguments");
  std::vector<const uint64_t*> all;
  for (int k = 0; k < n_plus; ++k) all.push_back(plus[k]);
  for (int k = 0; k < n_minus; ++k) all.push_back(minus[k]);
  for (const uint64_t* p : all)
    if (p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15))
      return set_error(EW_ERR_INVALID_ARGUMENT,
                       "ew_block_verifier_create: arrays must be non-NULL and 16-byte aligned");
  auto* v = new ew_block_verifier();
  v->n_plus = n_plus;
  v->n_minus = n_minus;
  v->lo = lo;
  v->hi = hi;
  if (!all.empty()) {
    cudaError_t e = cudaMalloc(&v->d_ptrs, all.size() * sizeof(void*));
    if (e == cudaSuccess)
      e = cudaMemcpy(v->d_ptrs, all.data(), all.size() * sizeof(void*), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      if (v->d_ptrs) cudaFree(v->d_ptrs);
      delete v;
      return cuda_status(e, "ew_block_verifier_create");
    }
  }
  *out = v;
  return EW_OK;
}

int ew_block_verifier_run(const ew_block_verifier* v, uint32_t* bad_count, ew_stream_t stream) {
  if (v == nullptr || bad_count == nullptr)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_block_verifier_run: NULL argument");
  EW_CUDA_TRY(cudaMemsetAsync(bad_count, 0, sizeof(uint32_t), (cudaStream_t)stream));
  const int64_t pairs = (v->hi - v->lo) / 2;
  if (pairs == 0 || v->n_plus + v->n_minus == 0) return EW_OK;
  const int grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>((pairs + 255) / 256, 4 * static_cast<int64_t>(num_sms()))));
  conservation_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(v->d_ptrs, v->n_plus, v->n_minus,
                                                              v->lo, v->hi, bad_count);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

void ew_block_verifier_free(ew_block_verifier* v) {
  if (v == nullptr) return;
  if (v->d_ptrs) cudaFree(v->d_ptrs);
  delete v;
}

}  // extern "C"
