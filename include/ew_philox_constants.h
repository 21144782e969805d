/* Philox-4x64-10 parameters shared by the host draws (elaskit::draw) and the
 * sm_100a mask kernel.  Values are the reference's (rng.cpp:8-14); the
 * counter layout {block, sample_id, (layer<<32)|op, 0} and the key
 * {seed, EW_PHILOX_KEY_DOMAIN} follow rng.cpp:40-48.  Usable from C, C++ and
 * CUDA device code. */
#ifndef EW_PHILOX_CONSTANTS_H
#define EW_PHILOX_CONSTANTS_H

#include <stdint.h>

#ifdef __CUDACC__
#define EW_HD __host__ __device__ __forceinline__
#else
#define EW_HD static inline
#endif

#define EW_PHILOX_ROUNDS 10
#define EW_PHILOX_M0 0xD2E7470EE14C6C93ULL
#define EW_PHILOX_M1 0xCA5A826395121157ULL
#define EW_PHILOX_W0 0x9E3779B97F4A7C15ULL
#define EW_PHILOX_W1 0xBB67AE8584CAA73BULL
#define EW_PHILOX_KEY_DOMAIN 0x454C41534B495431ULL

/* third counter word */
EW_HD uint64_t ew_philox_lane(uint32_t layer_id, uint32_t op_index) {
  return ((uint64_t)layer_id << 32) | (uint64_t)op_index;
}

/* 53-bit mantissa draw in [0,1) (reference: rng.cpp:51) */
EW_HD double ew_philox_unit(uint64_t word) {
  return (double)(word >> 11) * 0x1.0p-53;
}

/* Dropout rule of the reference toy step (sim.cpp:926-928): the element is
 * dropped iff u < keep_probability.  Because u = (w>>11) * 2^-53 exactly,
 * that is (w>>11) < ceil(keep * 2^53) in integers, which is what the device
 * kernel evaluates.  Returns the integer threshold; keep >= 1 drops all. */
EW_HD uint64_t ew_drop_threshold(double keep_probability) {
  if (!(keep_probability > 0.0)) return 0;               /* never dropped */
  if (keep_probability >= 1.0) return (1ULL << 53);      /* always dropped */
  double t = keep_probability * 9007199254740992.0;      /* exact: x * 2^53 */
  uint64_t ti = (uint64_t)t;                             /* floor, t < 2^53 */
  return ((double)ti == t) ? ti : ti + 1;                /* ceil */
}

#endif /* EW_PHILOX_CONSTANTS_H */
