// (c) Philox-4x64-10 dropout masks keyed by global sample id.
//
// The reference resharding of RNG is metadata only (reshard_rng, rng.cpp:73-97)
// because draw() is keyed by (seed, sample, layer, op) and nothing about DP/PP
// placement (rng.cpp:38-53).  This kernel generates the masks the reference
// toy step derives from draw() (sim.cpp:917-928) for any slice of the global
// sample range, so a rank generates exactly its own samples after a reshape
// with zero communication.  It is INT-ALU bound: 20 64x64->128 products per
// 4-element Philox block.  Each product is one 9-instruction IMAD chain with
// the multiplier halves as immediates; the first round's c2 product and the
// c3 = 0 word are constant per stream and hoisted out of the per-block loop.
#include <algorithm>

#include "ew_device.cuh"
#include "ew_philox_constants.h"

namespace ew {
namespace {

// (hi, lo) = a * b for a compile-time multiplier a.  The fmaheavy pipe is
// the limiter (ncu: 88.5 % busy with a hand-written 9-instruction mad.cc
// chain); letting ptxas lower mul.hi.u64 / mul.lo.u64 with the immediate
// halves folds the carries into IMAD.WIDE.U32.X and costs ~5 IMAD-class ops
// per product (tools/microbench/philox_variants.cu: 100 vs 87 G blocks/s).
template <uint64_t A>
__device__ __forceinline__ void mulhilo_c(uint64_t b, uint64_t& hi, uint64_t& lo) {
  hi = __umul64hi(A, b);
  lo = A * b;
}

struct Stream {
  uint64_t k0;        // seed
  uint64_t sample;    // counter word 1
  uint64_t lane;      // counter word 2
  uint64_t r0_hi1;    // round-0 M1*lane, hoisted
  uint64_t r0_lo1;
};

__device__ __forceinline__ Stream make_stream(uint64_t seed, uint64_t sample, uint64_t lane) {
  Stream s;
  s.k0 = seed;
  s.sample = sample;
  s.lane = lane;
  mulhilo_c<EW_PHILOX_M1>(lane, s.r0_hi1, s.r0_lo1);
  return s;
}

// philox4x64(counter = {block, sample, lane, 0}, key = {seed, KEY_DOMAIN})
__device__ __forceinline__ void philox_block(const Stream& s, uint64_t block, uint64_t out[4]) {
  uint64_t k0 = s.k0, k1 = EW_PHILOX_KEY_DOMAIN;
  uint64_t h0, l0;
  mulhilo_c<EW_PHILOX_M0>(block, h0, l0);
  // round 0 with c1 = sample, c2 = lane (hoisted product), c3 = 0
  uint64_t c0 = s.r0_hi1 ^ s.sample ^ k0;
  uint64_t c1 = s.r0_lo1;
  uint64_t c2 = h0 ^ k1;
  uint64_t c3 = l0;
#pragma unroll
  for (int r = 1; r < EW_PHILOX_ROUNDS; ++r) {
    k0 += EW_PHILOX_W0;
    k1 += EW_PHILOX_W1;
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo_c<EW_PHILOX_M0>(c0, hi0, lo0);
    mulhilo_c<EW_PHILOX_M1>(c2, hi1, lo1);
    const uint64_t n0 = hi1 ^ c1 ^ k0;
    const uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// One thread -> one 32-bit mask word = 8 Philox blocks of one sample.
__global__ void __launch_bounds__(256) mask_kernel(uint64_t seed, uint64_t sample_lo,
                                                   int64_t n_samples, uint64_t lane,
                                                   int64_t n_elems, int64_t words_per_row,
                                                   uint64_t threshold, uint32_t* __restrict__ bits) {
  const int64_t total = n_samples * words_per_row;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (w >= total) return;
  // (row, col) advanced by the grid stride: one 64-bit division per thread,
  // not one per word (a 64-bit divide is ~5 % of a word's 160-product budget)
  int64_t row = w / words_per_row, col = w - row * words_per_row;
  const int64_t srow = stride / words_per_row, scol = stride - srow * words_per_row;
  // the lane product of round 0 is the same for every word of the launch
  Stream s = make_stream(seed, sample_lo, lane);
  for (; w < total; w += stride, row += srow, col += scol) {
    if (col >= words_per_row) {
      col -= words_per_row;
      ++row;
    }
    // sample ids wrap mod 2^64 like the reference's uint64 RngKey::sample_id
    s.sample = sample_lo + static_cast<uint64_t>(row);
    const int64_t e0 = col * 32;
    const int nvalid = static_cast<int>(min((int64_t)32, n_elems - e0));
    uint32_t word = 0;
    if (nvalid == 32) {  // every word but a row's last: no per-element checks
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        uint64_t out[4];
        philox_block(s, static_cast<uint64_t>(col * 8 + b + 1), out);
#pragma unroll
        for (int i = 0; i < 4; ++i) word |= static_cast<uint32_t>(out[i] >= threshold) << (4 * b + i);
      }
      bits[w] = word;
      continue;
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      if (4 * b < nvalid) {
        uint64_t out[4];
        philox_block(s, static_cast<uint64_t>(col * 8 + b + 1), out);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          // dropped iff u < keep  <=>  (w >> 11) < threshold  <=>  w < threshold << 11
          // (the host passes threshold << 11, or ~0 with none_kept for keep >= 1)
          const bool kept = out[i] >= threshold;
          if (4 * b + i < nvalid && kept) word |= 1u << (4 * b + i);
        }
      }
    }
    bits[w] = word;
  }
}

__global__ void uniform_kernel(uint64_t seed, uint64_t sample_lo, int64_t n_samples, uint64_t lane,
                               int64_t n_elems, double* __restrict__ out) {
  const int64_t blocks_per_row = (n_elems + 3) / 4;
  const int64_t total = n_samples * blocks_per_row;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= total) return;
  // (row, blk) advanced by the grid stride, as in mask_kernel
  int64_t row = t / blocks_per_row, blk = t - row * blocks_per_row;
  const int64_t srow = stride / blocks_per_row, sblk = stride - srow * blocks_per_row;
  Stream s = make_stream(seed, sample_lo, lane);
  for (; t < total; t += stride, row += srow, blk += sblk) {
    if (blk >= blocks_per_row) {
      blk -= blocks_per_row;
      ++row;
    }
    s.sample = sample_lo + static_cast<uint64_t>(row);
    uint64_t w[4];
    philox_block(s, static_cast<uint64_t>(blk + 1), w);
    for (int i = 0; i < 4; ++i) {
      const int64_t k = 4 * blk + i;
      if (k < n_elems) out[row * n_elems + k] = ew_philox_unit(w[i]);
    }
  }
}

__global__ void words_kernel(uint64_t seed, uint64_t sample, uint64_t lane, uint64_t block_lo,
                             int64_t n_blocks, uint64_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_blocks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const Stream s = make_stream(seed, sample, lane);
    uint64_t w[4];
    philox_block(s, block_lo + static_cast<uint64_t>(t), w);
    for (int i = 0; i < 4; ++i) out[4 * t + i] = w[i];
  }
}

int grid_for(int64_t work) {
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, cap)));
}

}  // namespace
}  // namespace ew

using namespace ew;

extern "C" {

int ew_philox_dropout_mask(uint64_t seed, uint64_t sample_lo, int64_t n_samples,
                           uint32_t layer_id, uint32_t op_index, int64_t n_elems,
                           double keep_probability, uint32_t* bits, ew_stream_t stream) {
  if (n_samples < 0 || n_elems < 0)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_philox_dropout_mask: negative extent");
  if (n_samples == 0 || n_elems == 0) return EW_OK;
  if (bits == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_philox_dropout_mask: NULL bits");
  const int64_t wpr = (n_elems + 31) / 32;
  const uint64_t t53 = ew_drop_threshold(keep_probability);
  if (t53 >= (1ULL << 53)) {  // keep >= 1: u < keep always -> every element dropped
    EW_CUDA_TRY(cudaMemsetAsync(bits, 0, n_samples * wpr * sizeof(uint32_t), (cudaStream_t)stream));
    return EW_OK;
  }
  const uint64_t thr = t53 << 11;  // compare the raw word, no shift per element
  mask_kernel<<<grid_for(n_samples * wpr), 256, 0, (cudaStream_t)stream>>>(
      seed, sample_lo, n_samples, ew_philox_lane(layer_id, op_index), n_elems, wpr, thr, bits);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

int ew_philox_uniforms(uint64_t seed, uint64_t sample_lo, int64_t n_samples, uint32_t layer_id,
                       uint32_t op_index, int64_t n_elems, double* out, ew_stream_t stream) {
  if (n_samples < 0 || n_elems < 0)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_philox_uniforms: negative extent");
  if (n_samples == 0 || n_elems == 0) return EW_OK;
  if (out == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_philox_uniforms: NULL out");
  uniform_kernel<<<grid_for(n_samples * ((n_elems + 3) / 4)), 256, 0, (cudaStream_t)stream>>>(
      seed, sample_lo, n_samples, ew_philox_lane(layer_id, op_index), n_elems, out);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

int ew_philox_words(uint64_t seed, uint64_t sample_id, uint32_t layer_id, uint32_t op_index,
                    uint64_t block_lo, int64_t n_blocks, uint64_t* out, ew_stream_t stream) {
  if (n_blocks < 0) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_philox_words: negative count");
  if (n_blocks == 0) return EW_OK;
  if (out == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_philox_words: NULL out");
  words_kernel<<<grid_for(n_blocks), 256, 0, (cudaStream_t)stream>>>(
      seed, sample_id, ew_philox_lane(layer_id, op_index), block_lo, n_blocks, out);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

}  // extern "C"
