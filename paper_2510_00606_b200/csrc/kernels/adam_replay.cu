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

template <int kDepth>
__global__ void __launch_bounds__(256) adam_kernel(const float* __restrict__ grad,
                                                   float* __restrict__ master,
                                                   float* __restrict__ exp_avg,
                                                   float* __restrict__ exp_avg_sq,
                                                   uint16_t* __restrict__ param, int64_t n,
                                                   AdamScalars s) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(grad);
  float4* p4 = reinterpret_cast<float4*>(master);
  float4* m4 = reinterpret_cast<float4*>(exp_avg);
  float4* v4 = reinterpret_cast<float4*>(exp_avg_sq);
  uint2* b4 = reinterpret_cast<uint2*>(param);
  // kDepth independent groups per thread: the gradient may come from peer
  // HBM, so keep several NVLink loads in flight before the first use.
  // Measured at N=4 (tools/replay_sweep.sh): depth 1-3 and 4-16 CTAs/SM all
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
      __stcs(p4 + i, make_float4(e0.p, e1.p, e2.p, e3.p));
      __stcs(m4 + i, make_float4(e0.m, e1.m, e2.m, e3.m));
      __stcs(v4 + i, make_float4(e0.v, e1.v, e2.v, e3.v));
      __stcs(b4 + i, make_uint2(b0 | (b1 << 16), b2 | (b3 << 16)));
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
  }
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
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

int ew_adam_step(const float* grad, float* master, float* exp_avg, float* exp_avg_sq,
                 uint16_t* param_bf16, int64_t n, const ew_adam_hyper* hyper, int64_t step,
                 ew_stream_t stream) {
  if (n < 0 || (n > 0 && (!grad || !master || !exp_avg || !exp_avg_sq || !param_bf16)))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_adam_step: bad arguments");
  const auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!a16(grad) || !a16(master) || !a16(exp_avg) || !a16(exp_avg_sq) || (reinterpret_cast<uintptr_t>(param_bf16) & 7))
    return set_error(EW_ERR_INVALID_ARGUMENT,
                     "ew_adam_step: fp32 arrays must be 16-byte, bf16 array 8-byte aligned");
  float sc[8];
  if (int st = ew_adam_scalars(hyper, step, sc)) return st;
  if (n == 0) return EW_OK;
  const AdamScalars s{sc[0], sc[1], sc[2], sc[3], sc[4], sc[5], sc[6], sc[7]};
  const int64_t n4 = n / 4;
  const int64_t want = std::max<int64_t>(1, (std::max<int64_t>(n4, n - 4 * n4) + 255) / 256);
  const int grid = static_cast<int>(std::min<int64_t>(want, env_int("EW_ADAM_CTAS_PER_SM", 8) * num_sms()));
  const int depth = env_int("EW_ADAM_DEPTH", 2);
  const auto k = depth >= 4 ? adam_kernel<4> : depth == 3 ? adam_kernel<3> : depth == 1 ? adam_kernel<1> : adam_kernel<2>;
  k<<<grid, 256, 0, (cudaStream_t)stream>>>(grad, master, exp_avg, exp_avg_sq, param_bf16, n, s);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

}  // extern "C"
