// Ring-replica maintenance by optimizer replay.
//
// The paper backs up member (i+1)'s optimizer partition on member i: the
// owner sends only its reduced gradient shard (4 B/param instead of the
// 14 B/param of a mixed-precision Adam state, "at least 4x" less traffic)
// and the holder replays the Adam step into its replica (
// modelled by SnapshotTimeline, param_fabric.hpp:86-96).  The paper keeps the
// replica in host memory and steps it on the CPU; with 180 GB of HBM the
// holder keeps it in HBM and replays the step on its own GPU, reading the
// owner's gradient shard straight out of the owner's HBM over NVLink (a CUDA
// IPC peer pointer) inside the same kernel: pull and update are one pass.
//
// Bit-exactness: the owner runs this same kernel as its own ZeRO optimizer
// step, every operation is an explicitly rounded IEEE op (no contraction
// freedom), and the per-step scalars are derived once on the host, so the
// replica stays byte-identical to the owner's state and the owner's checksum
// rows verify it (kernel (a)).  oracle/ew_oracle.c restates the same update.
//
// State of one shard (n parameters) in HBM, structure of arrays, each array
// 256-byte aligned by the caller: fp32 master weights, fp32 exp_avg, fp32
// exp_avg_sq, bf16 parameters (the copy the forward pass reads).  Traffic per
// parameter: 4 B gradient (NVLink on the holder) + 12 B read + 14 B written.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "ew_device.cuh"

namespace ew {
namespace {

struct AdamScalars {
  float beta1, one_minus_beta1, beta2, one_minus_beta2, eps, step_size, inv_sqrt_bc2, decay;
};

// Round-to-nearest-even fp32 -> bf16 bits; NaN -> 0x7FC0 (same rule as the
// oracle's ew_oracle_bf16).
__device__ __forceinline__ uint32_t bf16_bits(float f) {
  const uint32_t u = __float_as_uint(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FC0u;
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}

struct Elem {
  float p, m, v;
};

__device__ __forceinline__ uint32_t adam_elem(const AdamScalars& s, float g, Elem& e) {
  const float m1 = __fmaf_rn(s.beta1, e.m, __fmul_rn(s.one_minus_beta1, g));
  const float v1 = __fmaf_rn(s.beta2, e.v, __fmul_rn(__fmul_rn(s.one_minus_beta2, g), g));
  const float denom = __fadd_rn(__fmul_rn(__fsqrt_rn(v1), s.inv_sqrt_bc2), s.eps);
  const float p1 = __fmaf_rn(-s.step_size, __fdiv_rn(m1, denom), __fmul_rn(e.p, s.decay));
  e.p = p1;
  e.m = m1;
  e.v = v1;
  return bf16_bits(p1);
}

// Checksum rows of the state's byte image fused into the step (kernel (a)'s
// spec: per block b, s0 = sum w_i, s1 = sum (i+1) w_i over the image's u64
// words, i the word index from the image base).  Each lane contributes the
// words it stores; the warp reduces when all 32 lanes fall in one block
// (the common case) and lane 0 adds the pair into the block's row.
struct RowSink {
  const uint8_t* base;           // state image base (global offset 0)
  unsigned long long* rows;      // [n_rows][2], zeroed before the launch
  int shift;                     // log2 block bytes
};

__device__ __forceinline__ void row_add(const RowSink& k, const void* at, uint64_t w0,
                                        uint64_t w1) {
  const int64_t off = reinterpret_cast<const uint8_t*>(at) - k.base;
  const uint64_t j = static_cast<uint64_t>(off) >> 3;
  uint64_t a = w0 + w1, b = (j + 1) * w0 + (j + 2) * w1;  // w1 = 0 for 8-byte stores
  const int64_t row = off >> k.shift;
  const int64_t row0 = __shfl_sync(0xffffffffu, row, 0);
  if (__all_sync(0xffffffffu, row == row0)) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(k.rows + 2 * row, static_cast<unsigned long long>(a));
      atomicAdd(k.rows + 2 * row + 1, static_cast<unsigned long long>(b));
    }
  } else {
    atomicAdd(k.rows + 2 * row, static_cast<unsigned long long>(a));
    atomicAdd(k.rows + 2 * row + 1, static_cast<unsigned long long>(b));
  }
}

__device__ __forceinline__ uint64_t lo64(float4 v) {
  return static_cast<uint64_t>(__float_as_uint(v.x)) |
         (static_cast<uint64_t>(__float_as_uint(v.y)) << 32);
}
__device__ __forceinline__ uint64_t hi64(float4 v) {
  return static_cast<uint64_t>(__float_as_uint(v.z)) |
         (static_cast<uint64_t>(__float_as_uint(v.w)) << 32);
}

template <int kDepth, bool kRows>
__global__ void __launch_bounds__(256) adam_kernel(const float* __restrict__ grad,
                                                   float* __restrict__ master,
                                                   float* __restrict__ exp_avg,
                                                   float* __restrict__ exp_avg_sq,
                                                   uint16_t* __restrict__ param, int64_t n,
                                                   AdamScalars s, RowSink sink) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(grad);
  float4* p4 = reinterpret_cast<float4*>(master);
  float4* m4 = reinterpret_cast<float4*>(exp_avg);
  float4* v4 = reinterpret_cast<float4*>(exp_avg_sq);
  uint2* b4 = reinterpret_cast<uint2*>(param);
  // kDepth independent groups per thread: the gradient may come from peer
  // HBM, so keep several NVLink loads in flight before the first use.
  // Measured at N=4 (tools/replay_sweep.sh, r01): depth 1-3 and 4-16 CTAs/SM all
  // give 5.3 ms for the 7B shard (636 GB/s of gradient over NVLink while the
  // holder's own HBM streams 26 B/param); depth 4 spills occupancy (5.8 ms);
  // a TMA-staged gradient ring measured 5.4-5.6 ms and was dropped.
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n4;
       i0 += kDepth * stride) {
    float4 g[kDepth], p[kDepth], m[kDepth], v[kDepth];
#pragma unroll
    for (int d = 0; d < kDepth; ++d) {
      const int64_t i = i0 + d * stride;
      if (i < n4) {
        g[d] = __ldcs(g4 + i);
        p[d] = __ldcs(p4 + i);
        m[d] = __ldcs(m4 + i);
        v[d] = __ldcs(v4 + i);
      }
    }
#pragma unroll
    for (int d = 0; d < kDepth; ++d) {
      const int64_t i = i0 + d * stride;
      if (i >= n4) continue;
      Elem e0{p[d].x, m[d].x, v[d].x}, e1{p[d].y, m[d].y, v[d].y};
      Elem e2{p[d].z, m[d].z, v[d].z}, e3{p[d].w, m[d].w, v[d].w};
      const uint32_t b0 = adam_elem(s, g[d].x, e0), b1 = adam_elem(s, g[d].y, e1);
      const uint32_t b2 = adam_elem(s, g[d].z, e2), b3 = adam_elem(s, g[d].w, e3);
      const float4 np4 = make_float4(e0.p, e1.p, e2.p, e3.p);
      const float4 nm4 = make_float4(e0.m, e1.m, e2.m, e3.m);
      const float4 nv4 = make_float4(e0.v, e1.v, e2.v, e3.v);
      const uint2 nb = make_uint2(b0 | (b1 << 16), b2 | (b3 << 16));
      __stcs(p4 + i, np4);
      __stcs(m4 + i, nm4);
      __stcs(v4 + i, nv4);
      __stcs(b4 + i, nb);
      if (kRows) {
        // warp-uniform here only if every lane has a valid i: the tail
        // iteration (i >= n4 on some lanes) takes the per-lane path below
        if (__activemask() == 0xffffffffu) {
          row_add(sink, p4 + i, lo64(np4), hi64(np4));
          row_add(sink, m4 + i, lo64(nm4), hi64(nm4));
          row_add(sink, v4 + i, lo64(nv4), hi64(nv4));
          row_add(sink, b4 + i, static_cast<uint64_t>(nb.x) | (static_cast<uint64_t>(nb.y) << 32), 0);
        } else {
          const uint8_t* at[4] = {reinterpret_cast<const uint8_t*>(p4 + i),
                                  reinterpret_cast<const uint8_t*>(m4 + i),
                                  reinterpret_cast<const uint8_t*>(v4 + i),
                                  reinterpret_cast<const uint8_t*>(b4 + i)};
          const uint64_t w0[4] = {lo64(np4), lo64(nm4), lo64(nv4),
                                  static_cast<uint64_t>(nb.x) | (static_cast<uint64_t>(nb.y) << 32)};
          const uint64_t w1[4] = {hi64(np4), hi64(nm4), hi64(nv4), 0};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int64_t off = at[q] - sink.base;
            const uint64_t j = static_cast<uint64_t>(off) >> 3;
            const int64_t row = off >> sink.shift;
            atomicAdd(sink.rows + 2 * row, static_cast<unsigned long long>(w0[q] + w1[q]));
            atomicAdd(sink.rows + 2 * row + 1,
                      static_cast<unsigned long long>((j + 1) * w0[q] + (j + 2) * w1[q]));
          }
        }
      }
    }
  }
  // scalar tail (n % 4 elements), one thread each
  const int64_t t = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) {
    Elem e{master[t], exp_avg[t], exp_avg_sq[t]};
    const uint32_t b = adam_elem(s, grad[t], e);
    master[t] = e.p;
    exp_avg[t] = e.m;
    exp_avg_sq[t] = e.v;
    param[t] = static_cast<uint16_t>(b);
    if (kRows) {  // partial words: a store's bytes shifted to their lane (linear)
      const void* at[4] = {master + t, exp_avg + t, exp_avg_sq + t, param + t};
      const uint64_t v[4] = {__float_as_uint(e.p), __float_as_uint(e.m), __float_as_uint(e.v), b};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t off = reinterpret_cast<const uint8_t*>(at[q]) - sink.base;
        const uint64_t x = v[q] << (8 * (off & 7));
        const uint64_t j = static_cast<uint64_t>(off) >> 3;
        const int64_t row = off >> sink.shift;
        atomicAdd(sink.rows + 2 * row, static_cast<unsigned long long>(x));
        atomicAdd(sink.rows + 2 * row + 1, static_cast<unsigned long long>((j + 1) * x));
      }
    }
  }
}



// Rows-fused step for block-aligned images: when every section starts on a
// checksum-block boundary, CTA c owns float4 groups [c*G, (c+1)*G) with
// G = block_bytes / 16, i.e. exactly block c of the master, exp_avg and
// exp_avg_sq sections and half of one block of the bf16 section.  Lanes
// accumulate their words' (s0, s1) in registers, the CTA reduces them once,
// and 8 global atomics deliver the CTA's share to its 4 rows.
__global__ void __launch_bounds__(256) adam_rows_kernel(
    const float* __restrict__ grad, float* __restrict__ master, float* __restrict__ exp_avg,
    float* __restrict__ exp_avg_sq, uint16_t* __restrict__ param, int64_t n4, AdamScalars s,
    RowSink sink) {
  const int64_t G = (int64_t{1} << sink.shift) >> 4;
  const int64_t f0 = blockIdx.x * G;
  const int64_t f1 = min(f0 + G, n4);
  const float4* g4 = reinterpret_cast<const float4*>(grad);
  float4* p4 = reinterpret_cast<float4*>(master);
  float4* m4 = reinterpret_cast<float4*>(exp_avg);
  float4* v4 = reinterpret_cast<float4*>(exp_avg_sq);
  uint2* b4 = reinterpret_cast<uint2*>(param);
  // word index of group f0's first word in each section
  const uint64_t w_p = static_cast<uint64_t>(reinterpret_cast<const uint8_t*>(p4 + f0) - sink.base) >> 3;
  const uint64_t w_m = static_cast<uint64_t>(reinterpret_cast<const uint8_t*>(m4 + f0) - sink.base) >> 3;
  const uint64_t w_v = static_cast<uint64_t>(reinterpret_cast<const uint8_t*>(v4 + f0) - sink.base) >> 3;
  const uint64_t w_b = static_cast<uint64_t>(reinterpret_cast<const uint8_t*>(b4 + f0) - sink.base) >> 3;
  uint64_t a[4] = {0, 0, 0, 0}, c[4] = {0, 0, 0, 0};
  for (int64_t i0 = f0 + threadIdx.x; i0 < f1; i0 += 2 * blockDim.x) {
    float4 g[2], p[2], m[2], v[2];
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      const int64_t i = i0 + d * blockDim.x;
      if (i < f1) {
        g[d] = __ldcs(g4 + i);
        p[d] = __ldcs(p4 + i);
        m[d] = __ldcs(m4 + i);
        v[d] = __ldcs(v4 + i);
      }
    }
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      const int64_t i = i0 + d * blockDim.x;
      if (i >= f1) continue;
      Elem e0{p[d].x, m[d].x, v[d].x}, e1{p[d].y, m[d].y, v[d].y};
      Elem e2{p[d].z, m[d].z, v[d].z}, e3{p[d].w, m[d].w, v[d].w};
      const uint32_t b0 = adam_elem(s, g[d].x, e0), b1 = adam_elem(s, g[d].y, e1);
      const uint32_t b2 = adam_elem(s, g[d].z, e2), b3 = adam_elem(s, g[d].w, e3);
      const float4 np4 = make_float4(e0.p, e1.p, e2.p, e3.p);
      const float4 nm4 = make_float4(e0.m, e1.m, e2.m, e3.m);
      const float4 nv4 = make_float4(e0.v, e1.v, e2.v, e3.v);
      const uint2 nb = make_uint2(b0 | (b1 << 16), b2 | (b3 << 16));
      __stcs(p4 + i, np4);
      __stcs(m4 + i, nm4);
      __stcs(v4 + i, nv4);
      __stcs(b4 + i, nb);
      const uint64_t r = static_cast<uint64_t>(i - f0);
      uint64_t x0 = lo64(np4), x1 = hi64(np4);
      a[0] += x0 + x1;
      c[0] += (w_p + 2 * r + 1) * x0 + (w_p + 2 * r + 2) * x1;
      x0 = lo64(nm4), x1 = hi64(nm4);
      a[1] += x0 + x1;
      c[1] += (w_m + 2 * r + 1) * x0 + (w_m + 2 * r + 2) * x1;
      x0 = lo64(nv4), x1 = hi64(nv4);
      a[2] += x0 + x1;
      c[2] += (w_v + 2 * r + 1) * x0 + (w_v + 2 * r + 2) * x1;
      x0 = static_cast<uint64_t>(nb.x) | (static_cast<uint64_t>(nb.y) << 32);
      a[3] += x0;
      c[3] += (w_b + r + 1) * x0;
    }
  }
  // CTA reduction of the 8 sums (mod 2^64)
  __shared__ uint64_t red[8][8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
      c[q] += __shfl_xor_sync(0xffffffffu, c[q], o);
    }
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      red[warp][2 * q] = a[q];
      red[warp][2 * q + 1] = c[q];
    }
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    uint64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w][threadIdx.x];
    const int q = threadIdx.x >> 1;
    const uint64_t w0 = q == 0 ? w_p : q == 1 ? w_m : q == 2 ? w_v : w_b;
    const int64_t row = static_cast<int64_t>((w0 << 3) >> sink.shift);
    if (t) atomicAdd(sink.rows + 2 * row + (threadIdx.x & 1), static_cast<unsigned long long>(t));
  }
}

}  // namespace
}  // namespace ew

using namespace ew;

extern "C" {

int ew_adam_scalars(const ew_adam_hyper* h, int64_t step, float* out8) {
  if (h == nullptr || out8 == nullptr || step < 1)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_adam_scalars: bad arguments (step >= 1)");
  if (!(h->beta1 >= 0.0 && h->beta1 < 1.0 && h->beta2 >= 0.0 && h->beta2 < 1.0 && h->eps > 0.0))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_adam_scalars: betas in [0,1), eps > 0");
  // torch.optim.AdamW semantics, scalars derived in fp64 and rounded once
  const double bc1 = 1.0 - std::pow(h->beta1, static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(h->beta2, static_cast<double>(step));
  out8[0] = static_cast<float>(h->beta1);
  out8[1] = static_cast<float>(1.0 - h->beta1);
  out8[2] = static_cast<float>(h->beta2);
  out8[3] = static_cast<float>(1.0 - h->beta2);
  out8[4] = static_cast<float>(h->eps);
  out8[5] = static_cast<float>(h->lr / bc1);
  out8[6] = static_cast<float>(1.0 / std::sqrt(bc2));
  out8[7] = static_cast<float>(1.0 - h->lr * h->weight_decay);
  return EW_OK;
}

static int adam_launch(const float* grad, float* master, float* exp_avg, float* exp_avg_sq,
                       uint16_t* param_bf16, int64_t n, const ew_adam_hyper* hyper,
                       int64_t step, const RowSink* sink, ew_stream_t stream) {
  if (n < 0 || (n > 0 && (!grad || !master || !exp_avg || !exp_avg_sq || !param_bf16)))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_adam_step: bad arguments");
  const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!a16(grad) || !a16(master) || !a16(exp_avg) || !a16(exp_avg_sq) ||
      (reinterpret_cast<uintptr_t>(param_bf16) & 7))
    return set_error(EW_ERR_INVALID_ARGUMENT,
                     "ew_adam_step: fp32 arrays must be 16-byte, bf16 array 8-byte aligned");
  float sc[8];
  if (int st = ew_adam_scalars(hyper, step, sc)) return st;
  if (n == 0) return EW_OK;
  const AdamScalars s{sc[0], sc[1], sc[2], sc[3], sc[4], sc[5], sc[6], sc[7]};
  const int64_t n4 = n / 4;
  const int64_t want = std::max<int64_t>(1, (std::max<int64_t>(n4, n - 4 * n4) + 255) / 256);
  const int grid = static_cast<int>(std::min<int64_t>(want, 8 * num_sms()));
  if (sink != nullptr) {
    const int64_t block = int64_t{1} << sink->shift;
    const auto aligned = [&](const void* q) {
      return ((static_cast<const uint8_t*>(q) - sink->base) & (block - 1)) == 0;
    };
    const bool fast = aligned(master) && aligned(exp_avg) && aligned(exp_avg_sq) &&
                      aligned(param_bf16);
    if (fast && n4 > 0) {
      adam_rows_kernel<<<static_cast<unsigned>((n4 + (block >> 4) - 1) / (block >> 4)), 256, 0,
                         (cudaStream_t)stream>>>(grad, master, exp_avg, exp_avg_sq, param_bf16,
                                                 n4, s, *sink);
      EW_CUDA_TRY(cudaGetLastError());
      if (n > 4 * n4) {  // < 4 tail elements: partial-word contributions per lane
        const int64_t t = 4 * n4;
        adam_kernel<1, true><<<1, 32, 0, (cudaStream_t)stream>>>(
            grad + t, master + t, exp_avg + t, exp_avg_sq + t, param_bf16 + t, n - t, s, *sink);
      }
    } else {  // sections not block-aligned: warp-reduced atomics per store
      adam_kernel<2, true><<<grid, 256, 0, (cudaStream_t)stream>>>(
          grad, master, exp_avg, exp_avg_sq, param_bf16, n, s, *sink);
    }
  } else
    adam_kernel<2, false><<<grid, 256, 0, (cudaStream_t)stream>>>(
        grad, master, exp_avg, exp_avg_sq, param_bf16, n, s, RowSink{});
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

int ew_adam_step(const float* grad, float* master, float* exp_avg, float* exp_avg_sq,
                 uint16_t* param_bf16, int64_t n, const ew_adam_hyper* hyper, int64_t step,
                 ew_stream_t stream) {
  return adam_launch(grad, master, exp_avg, exp_avg_sq, param_bf16, n, hyper, step, nullptr,
                     stream);
}

int ew_adam_step_rows(const float* grad, float* master, float* exp_avg, float* exp_avg_sq,
                      uint16_t* param_bf16, int64_t n, const ew_adam_hyper* hyper, int64_t step,
                      const void* image_base, int64_t image_bytes, int64_t block_bytes,
                      uint64_t* rows, ew_stream_t stream) {
  if (image_base == nullptr || rows == nullptr || image_bytes < 0 || block_bytes < 4096 ||
      block_bytes > (1 << 20) || (block_bytes & (block_bytes - 1)))
    return set_error(EW_ERR_INVALID_ARGUMENT,
                     "ew_adam_step_rows: image, rows and a power-of-two block in [4 KiB, 1 MiB]");
  const auto inside = [&](const void* p, int64_t bytes) {
    const auto* b = static_cast<const uint8_t*>(image_base);
    const auto* q = static_cast<const uint8_t*>(p);
    return q >= b && q + bytes <= b + image_bytes;
  };
  if (n > 0 && !(inside(master, 4 * n) && inside(exp_avg, 4 * n) && inside(exp_avg_sq, 4 * n) &&
                 inside(param_bf16, 2 * n)))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_adam_step_rows: arrays outside the image");
  const int64_t n_rows = (image_bytes + block_bytes - 1) / block_bytes;
  EW_CUDA_TRY(cudaMemsetAsync(rows, 0, 16 * n_rows, (cudaStream_t)stream));
  int shift = 0;
  while ((int64_t{1} << shift) < block_bytes) ++shift;
  const RowSink sink{static_cast<const uint8_t*>(image_base),
                     reinterpret_cast<unsigned long long*>(rows), shift};
  return adam_launch(grad, master, exp_avg, exp_avg_sq, param_bf16, n, hyper, step, &sink,
                     stream);
}

__global__ void rows_diff_kernel(const unsigned long long* __restrict__ a,
                                 const unsigned long long* __restrict__ b, int64_t n_rows,
                                 unsigned int* __restrict__ bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned int local = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows; r += stride)
    local += (a[2 * r] != b[2 * r] || a[2 * r + 1] != b[2 * r + 1]) ? 1u : 0u;
  if (local) atomicAdd(bad, local);
}

int ew_rows_diff(const uint64_t* a, const uint64_t* b, int64_t n_rows, uint32_t* bad_count,
                 ew_stream_t stream) {
  if (n_rows < 0 || bad_count == nullptr || (n_rows > 0 && (!a || !b)))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_rows_diff: bad arguments");
  EW_CUDA_TRY(cudaMemsetAsync(bad_count, 0, sizeof(uint32_t), (cudaStream_t)stream));
  if (n_rows == 0) return EW_OK;
  const int grid = static_cast<int>(std::min<int64_t>((n_rows + 255) / 256, 4 * num_sms()));
  rows_diff_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const unsigned long long*>(a), reinterpret_cast<const unsigned long long*>(b),
      n_rows, reinterpret_cast<unsigned int*>(bad_count));
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

}  // extern "C"
