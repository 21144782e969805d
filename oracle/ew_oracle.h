/* ORACLE — CPU restatement of the per-step DP recovery path (test
 * infrastructure only; see ew_oracle.c for the rules of use). */
#ifndef EW_ORACLE_H
#define EW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

void ew_oracle_philox4x64(const uint64_t counter[4], const uint64_t key[2], uint64_t out[4]);
void ew_oracle_draw(uint64_t seed, uint64_t sample, uint32_t layer, uint32_t op, int64_t n,
                    double* out);
void ew_oracle_dropout_mask(uint64_t seed, uint64_t sample_lo, int64_t n_samples, uint32_t layer,
                            uint32_t op, int64_t n_elems, double keep, uint32_t* bits);

uint64_t ew_oracle_splitmix64(uint64_t x);
int64_t ew_oracle_num_rows(const int64_t* segs, int64_t n_segs, int64_t block_bytes);
int64_t ew_oracle_row_sums(const int64_t* segs, int64_t n_segs, int64_t block_bytes,
                           const uint8_t* buf, uint64_t* out);
void ew_oracle_block_sums_synthetic(uint64_t seed, int64_t total_bytes, int64_t block_bytes,
                                    uint64_t* out);
void ew_oracle_fill_synthetic(const int64_t* segs, int64_t n_segs, uint64_t seed, uint8_t* buf);

int64_t ew_oracle_interleaved(const int64_t* layer_bytes, int n_layers, const int* ranks_sorted,
                              int n_ranks, int* out_counts, int64_t* out_ivs);
int64_t ew_oracle_overlap(const int* s_ranks, const int* s_counts, int s_n, const int64_t* s_ivs,
                          const int* d_ranks, const int* d_counts, int d_n, const int64_t* d_ivs,
                          const int* failed, int n_failed, const int* ring, int n_ring,
                          int64_t* out, int64_t cap);

int64_t ew_oracle_snapshot_mt(const int64_t* segs, int64_t n_segs, int64_t block,
                              const uint8_t* live, uint8_t* snap, uint64_t* sums, int threads);
int64_t ew_oracle_verify_mt(const int64_t* segs, int64_t n_segs, int64_t block,
                            const uint8_t* buf, const uint64_t* expected, int threads);

int ew_oracle_fixed_point_bits(double absmax, int64_t total_units);
void ew_oracle_weighted_fixed(const double* w, const float* g, int n_units, int64_t dim,
                              int frac_bits, int64_t* acc);

uint16_t ew_oracle_bf16(float f);
void ew_oracle_memcpy_mt(const uint8_t* const* src, uint8_t* const* dst, const int64_t* bytes,
                         int64_t n, int threads);
void ew_oracle_draw_mt(uint64_t seed, uint64_t sample_lo, int64_t n_samples, uint32_t layer,
                       uint32_t op, int64_t n_per_sample, double* out, int threads);
void ew_oracle_weighted_average_mt(const double* w, const double* g, int n_units, int64_t dim,
                                   double* out, int threads);
void ew_oracle_adam_scalars(double lr, double b1, double b2, double eps, double wd, int64_t step,
                            float out8[8]);
void ew_oracle_adam_step(const float* grad, float* master, float* exp_avg, float* exp_avg_sq,
                         uint16_t* param, int64_t n, double lr, double b1, double b2, double eps,
                         double wd, int64_t step);

/* synthetic-state rows / whole-space block sums on T threads (no buffer) */
int64_t ew_oracle_rows_synthetic_mt(uint64_t seed, const int64_t* segs, int64_t n_segs,
                                    int64_t block, uint64_t* out, int threads);
void ew_oracle_block_sums_synthetic_mt(uint64_t seed, int64_t total_bytes, int64_t block,
                                       uint64_t* out, int threads);

void ew_oracle_fill_synthetic_mt(const int64_t* segs, int64_t n_segs, uint64_t seed,
                                 uint8_t* buf, int64_t total, int threads);

#ifdef __cplusplus
}
#endif

#endif
