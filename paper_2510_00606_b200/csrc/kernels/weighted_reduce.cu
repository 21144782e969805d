// (d) Gradient-scale-preserving weighted reduce across reshaped micro-batches.
//
// Reference: weighted_grad_average (dataflow.cpp:71-83) is an fp64 left fold
// acc[i] += w_j * g_j[i] whose result depends on the fold order; the toy step
// gets split invariance only by walking samples in one canonical order
// (sim.cpp:901-953, test_dataflow.cpp:97-122).  On B200 the fold crosses GPUs
// through NCCL, whose summation order changes with world size, so the device
// path quantises each contribution unit once to int64 fixed point:
//     q_u[i] = rint(w_u * (double)g_u[i] * 2^F)
// and sums integers (exact, associative).  Any split of the same units over
// any number of ranks yields bit-identical sums; F comes from a global absmax
// pre-pass (an NCCL max, itself split-invariant).  Error vs the fp64
// reference: <= U * 2^-(F+1) from rounding, plus one fp32 rounding of output.
// The fold kernel is HBM-bound: 4 bytes per unit-element in, 8 bytes out.
#include <algorithm>
#include <cmath>

#include "ew_device.cuh"

namespace ew {
namespace {

constexpr int kMaxUnits = 16;

struct Units {
  const float* p[kMaxUnits];
  double w[kMaxUnits];
  int n;
};

// max_{k,i} |w_k * g_k[i]| (fp64 products).  Rounding is monotone, so
// max_i fl(|w_k| |g_k[i]|) = fl(|w_k| max_i |g_k[i]|): the stream only needs
// max_i |g_k[i]|, an integer max over the fp32 bit patterns with the sign
// cleared (non-negative floats order like their bits; every NaN pattern lies
// above +inf, so a NaN propagates as the max).  16-byte loads, kDepth deep,
// one REDUX per warp; each CTA then scales by |w_k| in fp64 and folds into
// the global max with one 64-bit atomicMax per unit (non-negative doubles
// and +NaN order like their bits too).  32-byte (256-bit) loads: streaming
// kernels reach ~6.6 TB/s with them against ~5.7 TB/s with 128-bit pairs.
__global__ void __launch_bounds__(256) absmax_kernel(Units u, int64_t n,
                                                     unsigned long long* out_bits) {
  constexpr int kDepth = 2;  // 2 x 32 B in flight per thread per unit
  constexpr uint32_t kAbs = 0x7fffffffu;
  __shared__ uint32_t red[kMaxUnits][8];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int k = 0; k < u.n; ++k) {
    uint32_t m = 0;
    const float* p = u.p[k];
    int64_t done = 0;
    if ((reinterpret_cast<uintptr_t>(p) & 31) == 0) {
      const int64_t n8 = n / 8;
      for (int64_t i0 = t0; i0 < n8; i0 += kDepth * stride) {
        Vec32 x[kDepth];
#pragma unroll
        for (int d = 0; d < kDepth; ++d) {
          const int64_t i = i0 + d * stride;
          x[d] = i < n8 ? ld_stream32(p + 8 * i) : Vec32{{0, 0, 0, 0}};
        }
#pragma unroll
        for (int d = 0; d < kDepth; ++d)
#pragma unroll
          for (int w = 0; w < 4; ++w)
            m = max(m, max(static_cast<uint32_t>(x[d].w[w]) & kAbs,
                           static_cast<uint32_t>(x[d].w[w] >> 32) & kAbs));
      }
      done = 8 * n8;
    }
    const uint32_t* s = reinterpret_cast<const uint32_t*>(p);
    for (int64_t i = done + t0; i < n; i += stride) m = max(m, __ldcs(s + i) & kAbs);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = m;
  }
  __syncthreads();
  if (threadIdx.x < u.n) {
    const int k = threadIdx.x;
    uint32_t m = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) m = max(m, red[k][w]);
    const double v = fabs(fabs(u.w[k]) * static_cast<double>(__uint_as_float(m)));
    atomicMax(out_bits, static_cast<unsigned long long>(__double_as_longlong(v)));
  }
}

// Fixed-point bits computed on the device (ew_fixed_point_bits_async): the
// whole (d) step can then run without a host round trip (CUDA-graph
// capturable).  kBadBits marks a non-finite or negative absmax.
constexpr int kBadBits = -2147483647 - 1;

__device__ __forceinline__ double device_scale(const int* bits, double host_scale) {
  if (bits == nullptr) return host_scale;
  const int f = *bits;
  return f == kBadBits ? 0.0 : ldexp(1.0, f);  // a bad scale folds to zeros
}

__global__ void scale_kernel(const double* __restrict__ gmax, int64_t total_units,
                             int* __restrict__ bits) {
  const double m = *gmax;
  if (!isfinite(m) || m < 0) {
    *bits = kBadBits;
    return;
  }
  if (m == 0.0) {
    *bits = 0;
    return;
  }
  int e = 0;
  frexp(m, &e);  // m < 2^e
  int cu = 0;
  while ((int64_t{1} << cu) < total_units) ++cu;
  *bits = min(1000, 62 - e - cu);  // total_units * m * 2^F < 2^62, as ew_fixed_point_bits
}

// kPipe (3+ units per element): one group per thread, unit k+1's load
// issued before unit k's math.  There the fold is bound by the conversion
// pipe (F2F.F64.F32 + F2I.S64.F64, ~15/clk/SM measured) rather than HBM, and
// overlapping the next unit's latency with this unit's conversions is worth
// ~11 % at 4 and 8 units (tools/microbench/fold_variants.cu); at 1-2 units
// the two-deep unpipelined form streams faster.  Bounded to 4 CTAs/SM (64
// registers; the pipelined forms keep 8-16 B on the stack, measured faster
// than 80 registers at 3 CTAs/SM: tools/fold_sweep.py).  Unit loads carry no
// L2 evict-first hint: a unit buffer listed twice (config E's N = 1 leg)
// then re-reads from L2.
//
// Grids, % of the resident CTAs (tools/fold_grid_sweep.sh, 7B gradient): the
// write-heavy streams run best oversubscribed 1.6x (fold of one unit 12.7 vs
// 13.5 ms, dequant 12.5 vs 13.2 ms), the fold of two units and the
// read-only absmax at one wave, the pipelined fold at three waves.
constexpr int kFoldGrid1Pct = 160;     // 1 unit
constexpr int kFoldGridPct = 100;      // 2 units
constexpr int kFoldPipeGridPct = 300;  // 3+ units (pipelined)
constexpr int kAbsmaxGridPct = 100;
constexpr int kDequantGridPct = 160;

template <bool kAccumulate, bool kPipe>
__global__ void __launch_bounds__(256, 4) fold_kernel(Units u, int64_t n, double host_scale,
                                                   long long* __restrict__ acc,
                                                   const long long* __restrict__ addend,
                                                   const int* __restrict__ dev_bits) {
  const double scale = device_scale(dev_bits, host_scale);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n8 = n / 8;
  // 256-bit path: 8 elements per group, one 32-byte load per unit, two
  // 32-byte stores of the int64 sums
  bool vec_ok = ((reinterpret_cast<uintptr_t>(acc) | reinterpret_cast<uintptr_t>(addend)) & 31) == 0;
  for (int k = 0; k < u.n; ++k) vec_ok = vec_ok && ((reinterpret_cast<uintptr_t>(u.p[k]) & 31) == 0);
  if (vec_ok) {
    constexpr int kDepth = kPipe ? 1 : 2;  // independent 32-byte groups per thread
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n8;
         i0 += kDepth * stride) {
      auto load = [&](const float* p, Vec32 (&g)[kDepth]) {
#pragma unroll
        for (int d = 0; d < kDepth; ++d) {
          const int64_t i = i0 + d * stride;
          g[d] = i < n8 ? ld_nc32(p + 8 * i) : Vec32{{0, 0, 0, 0}};
        }
      };
      long long s[kDepth][8] = {};
      Vec32 g[kDepth];
      if (kPipe) load(u.p[0], g);
      for (int k = 0; k < u.n; ++k) {
        Vec32 next[kDepth];
        if (!kPipe)
          load(u.p[k], g);
        else if (k + 1 < u.n)
          load(u.p[k + 1], next);
        const double w = u.w[k];
#pragma unroll
        for (int d = 0; d < kDepth; ++d)
#pragma unroll
          for (int e = 0; e < 8; ++e)
            s[d][e] += __double2ll_rn((w * static_cast<double>(f32_of(g[d], e))) * scale);
        if (kPipe) {
#pragma unroll
          for (int d = 0; d < kDepth; ++d) g[d] = next[d];
        }
      }
#pragma unroll
      for (int d = 0; d < kDepth; ++d) {
        const int64_t i = i0 + d * stride;
        if (i >= n8) break;
        long long* dst = acc + 8 * i;
        if (kAccumulate) {
          const Vec32 a = ld_plain32(dst), b = ld_plain32(dst + 4);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            s[d][e] += static_cast<long long>(a.w[e]);
            s[d][4 + e] += static_cast<long long>(b.w[e]);
          }
        }
        if (addend != nullptr) {  // e.g. a migration's shadow-gradient payback
          const Vec32 a = ld_stream32(addend + 8 * i), b = ld_stream32(addend + 8 * i + 4);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            s[d][e] += static_cast<long long>(a.w[e]);
            s[d][4 + e] += static_cast<long long>(b.w[e]);
          }
        }
        Vec32 lo, hi;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          lo.w[e] = static_cast<uint64_t>(s[d][e]);
          hi.w[e] = static_cast<uint64_t>(s[d][4 + e]);
        }
        st_stream32(dst, lo);
        st_stream32(dst + 4, hi);
      }
    }
  }
  const int64_t start = vec_ok ? 8 * n8 : 0;
  for (int64_t i = start + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    long long s = kAccumulate ? acc[i] : 0;
    if (addend != nullptr) s += addend[i];
    for (int k = 0; k < u.n; ++k)
      s += __double2ll_rn((u.w[k] * static_cast<double>(u.p[k][i])) * scale);
    acc[i] = s;
  }
}

// out[i] = (T)((double)acc[i] * 2^-F): groups of 8 elements, two 32-byte
// loads and one 32-byte (fp32) or two (fp64) stores each, kDepth groups in
// flight per thread; scalar tail.
template <typename T>
__device__ __forceinline__ void store8(T* out, int64_t g, const double (&v)[8]);
template <>
__device__ __forceinline__ void store8<float>(float* out, int64_t g, const double (&v)[8]) {
  Vec32 o;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    o.w[k] = static_cast<uint64_t>(__float_as_uint(static_cast<float>(v[2 * k]))) |
             (static_cast<uint64_t>(__float_as_uint(static_cast<float>(v[2 * k + 1]))) << 32);
  st_stream32(out + 8 * g, o);
}
template <>
__device__ __forceinline__ void store8<double>(double* out, int64_t g, const double (&v)[8]) {
  Vec32 lo, hi;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    lo.w[k] = static_cast<uint64_t>(__double_as_longlong(v[k]));
    hi.w[k] = static_cast<uint64_t>(__double_as_longlong(v[4 + k]));
  }
  st_stream32(out + 8 * g, lo);
  st_stream32(out + 8 * g + 4, hi);
}

template <typename T>
__global__ void __launch_bounds__(256) dequant_kernel(const long long* __restrict__ acc, int64_t n,
                                                      double host_inv_scale, T* __restrict__ out,
                                                      const int* __restrict__ dev_bits) {
  const double inv_scale = dev_bits == nullptr ? host_inv_scale
                           : (*dev_bits == kBadBits ? 0.0 : ldexp(1.0, -*dev_bits));
  constexpr int kDepth = 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t done = 0;
  if (((reinterpret_cast<uintptr_t>(acc) | reinterpret_cast<uintptr_t>(out)) & 31) == 0) {
    const int64_t n8 = n / 8;
    for (int64_t g0 = t0; g0 < n8; g0 += kDepth * stride) {
      Vec32 x[kDepth][2];
#pragma unroll
      for (int d = 0; d < kDepth; ++d) {
        const int64_t g = g0 + d * stride;
        if (g < n8) {
          x[d][0] = ld_stream32(acc + 8 * g);
          x[d][1] = ld_stream32(acc + 8 * g + 4);
        }
      }
#pragma unroll
      for (int d = 0; d < kDepth; ++d) {
        const int64_t g = g0 + d * stride;
        if (g >= n8) break;
        double v[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[e] = static_cast<double>(static_cast<long long>(x[d][0].w[e])) * inv_scale;
          v[4 + e] = static_cast<double>(static_cast<long long>(x[d][1].w[e])) * inv_scale;
        }
        store8<T>(out, g, v);
      }
    }
    done = 8 * n8;
  }
  for (int64_t i = done + t0; i < n; i += stride)
    out[i] = static_cast<T>(static_cast<double>(acc[i]) * inv_scale);
}

int grid_for(int64_t work) {
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, cap)));
}

// Persistent grid for the 256-thread streaming kernels: every CTA resident
// (SMs x occupancy), so the grid-stride loops run in one wave.
int resident_grid(const void* kernel, int64_t work, int pct = 100) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0);
  const int64_t cap = std::max<int64_t>(
      1, static_cast<int64_t>(num_sms()) * std::max(1, per_sm) * pct / 100);
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, cap)));
}

int pack_units(const float* const* units, const double* weights, int n_units, int offset,
               Units& u) {
  u.n = std::min(kMaxUnits, n_units - offset);
  for (int k = 0; k < u.n; ++k) {
    if (units[offset + k] == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL unit pointer");
    u.p[k] = units[offset + k];
    u.w[k] = weights[offset + k];
  }
  for (int k = u.n; k < kMaxUnits; ++k) {
    u.p[k] = nullptr;
    u.w[k] = 0.0;
  }
  return EW_OK;
}

}  // namespace
}  // namespace ew

using namespace ew;

extern "C" {

int ew_weighted_absmax(const float* const* units, const double* weights, int n_units,
                       int64_t n_elems, double* out_max, ew_stream_t stream) {
  if (out_max == nullptr || n_units < 0 || n_elems < 0 || (n_units > 0 && (!units || !weights)))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_weighted_absmax: bad arguments");
  EW_CUDA_TRY(cudaMemsetAsync(out_max, 0, sizeof(double), (cudaStream_t)stream));
  for (int off = 0; off < n_units && n_elems > 0; off += kMaxUnits) {
    Units u;
    if (int st = pack_units(units, weights, n_units, off, u)) return st;
    absmax_kernel<<<resident_grid((const void*)absmax_kernel, (n_elems + 7) / 8, kAbsmaxGridPct), 256, 0,
                    (cudaStream_t)stream>>>(
        u, n_elems, reinterpret_cast<unsigned long long*>(out_max));
    EW_CUDA_TRY(cudaGetLastError());
  }
  return EW_OK;
}

int ew_fixed_point_bits(double global_absmax, int64_t total_units, int* frac_bits) {
  if (frac_bits == nullptr || total_units < 1)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_fixed_point_bits: bad arguments");
  if (!std::isfinite(global_absmax) || global_absmax < 0)
    return set_error(EW_ERR_INVALID_ARGUMENT, "gradient contains inf/nan");
  if (global_absmax == 0.0) {
    *frac_bits = 0;
    return EW_OK;
  }
  int e = 0;
  std::frexp(global_absmax, &e);  // absmax < 2^e
  int cu = 0;
  while ((int64_t{1} << cu) < total_units) ++cu;  // total_units <= 2^cu
  *frac_bits = std::min(1000, 62 - e - cu);       // U * absmax * 2^F < 2^62
  return EW_OK;
}

int ew_weighted_fold(const float* const* units, const double* weights, int n_units,
                     int64_t n_elems, int frac_bits, int64_t* acc, int accumulate,
                     ew_stream_t stream) {
  return ew_weighted_fold_addend(units, weights, n_units, n_elems, frac_bits, acc, accumulate,
                                 nullptr, stream);
}

}  // extern "C"

namespace ew {
namespace {

// fold with the scale 2^frac_bits, or 2^(*dev_bits) when dev_bits != NULL
int fold_impl(const float* const* units, const double* weights, int n_units, int64_t n_elems,
              int frac_bits, const int* dev_bits, int64_t* acc, int accumulate,
              const int64_t* addend, ew_stream_t stream) {
  if ((n_elems > 0 && acc == nullptr) || n_units < 0 || n_elems < 0 ||
      (n_units > 0 && (!units || !weights)))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_weighted_fold: bad arguments");
  if (dev_bits == nullptr && (frac_bits > 1000 || frac_bits < -1000))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_weighted_fold: frac_bits out of range");
  if (n_elems == 0) return EW_OK;
  const double scale = dev_bits == nullptr ? std::ldexp(1.0, frac_bits) : 0.0;
  if (n_units == 0) {
    if (!accumulate)
      EW_CUDA_TRY(cudaMemsetAsync(acc, 0, n_elems * sizeof(int64_t), (cudaStream_t)stream));
    return addend ? ew_payback_accumulate(acc, addend, n_elems, stream) : EW_OK;
  }
  for (int off = 0; off < n_units; off += kMaxUnits) {
    Units u;
    if (int st = pack_units(units, weights, n_units, off, u)) return st;
    long long* a = reinterpret_cast<long long*>(acc);
    const long long* add = off == 0 ? reinterpret_cast<const long long*>(addend) : nullptr;
    const bool accum = accumulate || off > 0;
    const bool pipe = u.n >= 3;
    const void* kern = accum ? (pipe ? (const void*)fold_kernel<true, true>
                                     : (const void*)fold_kernel<true, false>)
                             : (pipe ? (const void*)fold_kernel<false, true>
                                     : (const void*)fold_kernel<false, false>);
    // 64 registers x 256 threads: 4 resident CTAs/SM
    const int grid = resident_grid(kern, (n_elems + 7) / 8,
                                   pipe ? kFoldPipeGridPct : u.n == 1 ? kFoldGrid1Pct : kFoldGridPct);
    void* args[] = {&u, &n_elems, const_cast<double*>(&scale), &a, &add,
                    &dev_bits};
    EW_CUDA_TRY(cudaLaunchKernel(kern, grid, 256, args, 0, (cudaStream_t)stream));
    EW_CUDA_TRY(cudaGetLastError());
  }
  return EW_OK;
}

template <typename T>
int dequant_impl(const int64_t* acc, int64_t n, int frac_bits, const int* dev_bits, T* out,
                 ew_stream_t stream) {
  if ((n > 0 && (!acc || !out)) || n < 0)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_fixed_to_float/double: bad arguments");
  if (n == 0) return EW_OK;
  dequant_kernel<T><<<resident_grid((const void*)dequant_kernel<T>, (n + 7) / 8, kDequantGridPct), 256, 0,
                      (cudaStream_t)stream>>>(reinterpret_cast<const long long*>(acc), n,
                                              std::ldexp(1.0, -frac_bits), out, dev_bits);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

}  // namespace
}  // namespace ew

extern "C" {

int ew_weighted_fold_addend(const float* const* units, const double* weights, int n_units,
                            int64_t n_elems, int frac_bits, int64_t* acc, int accumulate,
                            const int64_t* addend, ew_stream_t stream) {
  return fold_impl(units, weights, n_units, n_elems, frac_bits, nullptr, acc, accumulate, addend,
                   stream);
}

int ew_fixed_point_bits_async(const double* global_absmax, int64_t total_units, int* frac_bits,
                              ew_stream_t stream) {
  if (global_absmax == nullptr || frac_bits == nullptr || total_units < 1)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_fixed_point_bits_async: bad arguments");
  scale_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(global_absmax, total_units, frac_bits);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

int ew_weighted_fold_dev(const float* const* units, const double* weights, int n_units,
                         int64_t n_elems, const int* frac_bits, int64_t* acc, int accumulate,
                         const int64_t* addend, ew_stream_t stream) {
  if (frac_bits == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL frac_bits");
  return fold_impl(units, weights, n_units, n_elems, 0, frac_bits, acc, accumulate, addend,
                   stream);
}

int ew_fixed_to_float_dev(const int64_t* acc, int64_t n, const int* frac_bits, float* out,
                          ew_stream_t stream) {
  if (frac_bits == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL frac_bits");
  return dequant_impl<float>(acc, n, 0, frac_bits, out, stream);
}

int ew_fixed_to_float(const int64_t* acc, int64_t n, int frac_bits, float* out,
                      ew_stream_t stream) {
  return dequant_impl<float>(acc, n, frac_bits, nullptr, out, stream);
}

int ew_fixed_to_double(const int64_t* acc, int64_t n, int frac_bits, double* out,
                       ew_stream_t stream) {
  return dequant_impl<double>(acc, n, frac_bits, nullptr, out, stream);
}

}  // extern "C"

namespace ew {
namespace {

__global__ void __launch_bounds__(256) payback_kernel(long long* __restrict__ acc,
                                                      const long long* __restrict__ payback,
                                                      int64_t n) {
  // 2 x 16 B per thread-iteration in flight; payback usually lives in peer HBM
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n2 = n / 2;
  const longlong2* p2 = reinterpret_cast<const longlong2*>(payback);
  longlong2* a2 = reinterpret_cast<longlong2*>(acc);
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n2; i0 += 2 * stride) {
    const int64_t i1 = i0 + stride;
    const longlong2 x0 = __ldcs(p2 + i0);
    const longlong2 y0 = a2[i0];
    longlong2 x1 = make_longlong2(0, 0), y1 = make_longlong2(0, 0);
    if (i1 < n2) {
      x1 = __ldcs(p2 + i1);
      y1 = a2[i1];
    }
    // two's-complement wrap, like the int64 NCCL sum
    a2[i0] = make_longlong2(static_cast<long long>(static_cast<unsigned long long>(y0.x) + static_cast<unsigned long long>(x0.x)),
                            static_cast<long long>(static_cast<unsigned long long>(y0.y) + static_cast<unsigned long long>(x0.y)));
    if (i1 < n2)
      a2[i1] = make_longlong2(static_cast<long long>(static_cast<unsigned long long>(y1.x) + static_cast<unsigned long long>(x1.x)),
                              static_cast<long long>(static_cast<unsigned long long>(y1.y) + static_cast<unsigned long long>(x1.y)));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1))
    acc[n - 1] = static_cast<long long>(static_cast<unsigned long long>(acc[n - 1]) +
                                        static_cast<unsigned long long>(payback[n - 1]));
}

}  // namespace
}  // namespace ew

extern "C" int ew_payback_accumulate(int64_t* acc, const int64_t* payback, int64_t n,
                                     ew_stream_t stream) {
  using namespace ew;
  if (n < 0 || (n > 0 && (!acc || !payback)))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_payback_accumulate: bad arguments");
  if ((reinterpret_cast<uintptr_t>(acc) | reinterpret_cast<uintptr_t>(payback)) & 15)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_payback_accumulate: buffers must be 16-byte aligned");
  if (n == 0) return EW_OK;
  const int grid = grid_for((n + 3) / 4);
  payback_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<long long*>(acc),
                                                         reinterpret_cast<const long long*>(payback), n);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}
