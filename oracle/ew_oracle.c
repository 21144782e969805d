/* ORACLE — CPU restatement of the per-step DP recovery path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline — never as the product path.
 *
 * Each function restates the reference algorithm it follows (file:line into
 * /root/reference/proj), written for clarity rather than speed and
 * independently of the B200 implementation:
 *   - Philox-4x64-10 / draw():  rng.cpp:8-53           (pinned: golden JSON)
 *   - dropout rule:            sim.cpp:917-928         (pinned: via draw())
 *   - interleaved ZeRO layout:  migration.cpp:73-77 + SURVEY §8(a) A4
 *   - overlap_matrix:           param_fabric.cpp:82-121 (pinned: oracle/_ref)
 *   - plan execution:           test_param_fabric.cpp:20-29 apply_plan, as bytes
 *   - fixed-point weighted fold: dataflow.cpp:71-83 re-based on int64 sums
 *   - per-block checksum:       NO reference code — PARITY UNPINNED; this file
 *     is the definition (ew_api.h "Checksum spec"), golden vectors under
 *     tests/golden/ are generated from it.
 */
#include "ew_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------- Philox (rng.cpp:8-36) ---------------- */

static const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
static const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
static const uint64_t KEY_DOMAIN = 0x454C41534B495431ULL; /* rng.cpp:14 */

void ew_oracle_philox4x64(const uint64_t counter[4], const uint64_t key[2], uint64_t out[4]) {
  uint64_t c0 = counter[0], c1 = counter[1], c2 = counter[2], c3 = counter[3];
  uint64_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    unsigned __int128 p0 = (unsigned __int128)M0 * c0;
    unsigned __int128 p1 = (unsigned __int128)M1 * c2;
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0;
    k1 += W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* rng.cpp:38-53: element k <- word k%4 of block 1 + k/4; u = (w >> 11) 2^-53 */
void ew_oracle_draw(uint64_t seed, uint64_t sample, uint32_t layer, uint32_t op, int64_t n,
                    double* out) {
  const uint64_t key[2] = {seed, KEY_DOMAIN};
  const uint64_t lane = ((uint64_t)layer << 32) | op;
  uint64_t w[4];
  for (int64_t k = 0; k < n; ++k) {
    if (k % 4 == 0) {
      const uint64_t ctr[4] = {1 + (uint64_t)(k / 4), sample, lane, 0};
      ew_oracle_philox4x64(ctr, key, w);
    }
    out[k] = (double)(w[k % 4] >> 11) * 0x1.0p-53;
  }
}

/* sim.cpp:926-928 literally: mask = u < keep ? 0 : 1/keep.  bit 1 = kept. */
void ew_oracle_dropout_mask(uint64_t seed, uint64_t sample_lo, int64_t n_samples, uint32_t layer,
                            uint32_t op, int64_t n_elems, double keep, uint32_t* bits) {
  const int64_t wpr = (n_elems + 31) / 32;
  double* u = (double*)malloc((size_t)(n_elems > 0 ? n_elems : 1) * sizeof(double));
  for (int64_t s = 0; s < n_samples; ++s) {
    uint32_t* row = bits + s * wpr;
    memset(row, 0, (size_t)wpr * 4);
    ew_oracle_draw(seed, sample_lo + (uint64_t)s, layer, op, n_elems, u);
    for (int64_t k = 0; k < n_elems; ++k)
      if (!(u[k] < keep)) row[k / 32] |= 1u << (k % 32);
  }
  free(u);
}

/* ---------------- per-block checksum (builder-defined) ---------------- */

uint64_t ew_oracle_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

int64_t ew_oracle_num_rows(const int64_t* segs, int64_t n_segs, int64_t block_bytes) {
  int64_t rows = 0;
  for (int64_t k = 0; k < n_segs; ++k) {
    const int64_t glo = segs[3 * k], len = segs[3 * k + 1];
    if (len > 0) rows += (glo + len - 1) / block_bytes - glo / block_bytes + 1;
  }
  return rows;
}

/* Rows in segment order, blocks ascending inside a segment.  For every
 * global word i touched by the row, w_i is assembled byte by byte from the
 * bytes the segment holds (others are zero); s0 += w_i, s1 += (i+1) w_i. */
int64_t ew_oracle_row_sums(const int64_t* segs, int64_t n_segs, int64_t block_bytes,
                           const uint8_t* buf, uint64_t* out) {
  int64_t r = 0;
  for (int64_t k = 0; k < n_segs; ++k) {
    const int64_t glo = segs[3 * k], len = segs[3 * k + 1], loff = segs[3 * k + 2];
    if (len <= 0) continue;
    for (int64_t b = glo / block_bytes; b <= (glo + len - 1) / block_bytes; ++b, ++r) {
      const int64_t lo = glo > b * block_bytes ? glo : b * block_bytes;
      const int64_t hi = (glo + len) < (b + 1) * block_bytes ? (glo + len) : (b + 1) * block_bytes;
      uint64_t s0 = 0, s1 = 0;
      for (int64_t i = lo / 8; i <= (hi - 1) / 8; ++i) {
        uint64_t w = 0;
        for (int j = 0; j < 8; ++j) {
          const int64_t g = 8 * i + j;
          if (g >= lo && g < hi) w |= (uint64_t)buf[loff + (g - glo)] << (8 * j);
        }
        s0 += w;
        s1 += (uint64_t)(i + 1) * w;
      }
      out[2 * r] = s0;
      out[2 * r + 1] = s1;
    }
  }
  return r;
}

/* Whole-space block sums of the synthetic state w_i = splitmix64(seed ^ i). */
void ew_oracle_block_sums_synthetic(uint64_t seed, int64_t total_bytes, int64_t block_bytes,
                                    uint64_t* out) {
  const int64_t n_blocks = (total_bytes + block_bytes - 1) / block_bytes;
  for (int64_t b = 0; b < n_blocks; ++b) {
    const int64_t lo = b * block_bytes;
    const int64_t hi = lo + block_bytes < total_bytes ? lo + block_bytes : total_bytes;
    uint64_t s0 = 0, s1 = 0;
    for (int64_t i = lo / 8; i <= (hi - 1) / 8; ++i) {
      uint64_t w = ew_oracle_splitmix64(seed ^ (uint64_t)i);
      if (8 * i + 8 > hi) w &= (hi - 8 * i) >= 8 ? ~0ULL : ((1ULL << (8 * (hi - 8 * i))) - 1);
      s0 += w;
      s1 += (uint64_t)(i + 1) * w;
    }
    out[2 * b] = s0;
    out[2 * b + 1] = s1;
  }
}

void ew_oracle_fill_synthetic(const int64_t* segs, int64_t n_segs, uint64_t seed, uint8_t* buf) {
  for (int64_t k = 0; k < n_segs; ++k) {
    const int64_t glo = segs[3 * k], len = segs[3 * k + 1], loff = segs[3 * k + 2];
    for (int64_t x = 0; x < len; ++x) {
      const int64_t g = glo + x;
      buf[loff + x] = (uint8_t)(ew_oracle_splitmix64(seed ^ (uint64_t)(g / 8)) >> (8 * (g % 8)));
    }
  }
}

/* ---------------- layouts and plans ---------------- */

/* migration.cpp:73-77 shard rule composed per SURVEY A4: for each layer, for
 * each rank index j (ranks ascending), [off + sz*j/D, off + sz*(j+1)/D) if
 * non-empty.  out_counts[j] intervals for ranks[j] (sorted), rows in out_ivs
 * grouped by rank.  Returns the number of intervals. */
int64_t ew_oracle_interleaved(const int64_t* layer_bytes, int n_layers, const int* ranks_sorted,
                              int n_ranks, int* out_counts, int64_t* out_ivs) {
  int64_t total = 0;
  for (int j = 0; j < n_ranks; ++j) out_counts[j] = 0;
  for (int j = 0; j < n_ranks; ++j) {
    int64_t off = 0;
    for (int l = 0; l < n_layers; ++l) {
      const int64_t sz = layer_bytes[l];
      const int64_t lo = off + sz * j / n_ranks, hi = off + sz * (j + 1) / n_ranks;
      if (hi > lo) {
        out_ivs[2 * total] = lo;
        out_ivs[2 * total + 1] = hi;
        ++total;
        ++out_counts[j];
      }
      off += sz;
    }
  }
  (void)ranks_sorted;
  return total;
}

typedef struct {
  int64_t src, dst, lo, hi, medium;
} row5;

static int cmp_lo(const void* a, const void* b) {
  const row5* x = (const row5*)a;
  const row5* y = (const row5*)b;
  return (x->lo > y->lo) - (x->lo < y->lo);
}

static int contains(const int* v, int n, int x) {
  for (int i = 0; i < n; ++i)
    if (v[i] == x) return 1;
  return 0;
}

/* param_fabric.cpp:82-121 as nested loops over (src interval, dst rank,
 * dst interval).  Preconditions (validate, ring) are the caller's; a dead
 * owner is sourced from the ring member before it (param_fabric.cpp:51-57).
 * Rows {src, dst, lo, hi, medium}.  Returns the entry count (or -1 if cap is
 * too small). */
int64_t ew_oracle_overlap(const int* s_ranks, const int* s_counts, int s_n, const int64_t* s_ivs,
                          const int* d_ranks, const int* d_counts, int d_n, const int64_t* d_ivs,
                          const int* failed, int n_failed, const int* ring, int n_ring,
                          int64_t* out, int64_t cap) {
  int64_t n = 0;
  int64_t si = 0;
  for (int a = 0; a < s_n; ++a) {
    const int owner = s_ranks[a];
    const int dead = contains(failed, n_failed, owner);
    int phys = owner;
    if (dead) {
      for (int k = 0; k < n_ring; ++k)
        if (ring[k] == owner) phys = ring[(k - 1 + n_ring) % n_ring];
    }
    for (int c = 0; c < s_counts[a]; ++c, ++si) {
      const int64_t slo = s_ivs[2 * si], shi = s_ivs[2 * si + 1];
      int64_t di = 0;
      for (int b = 0; b < d_n; ++b) {
        for (int e = 0; e < d_counts[b]; ++e, ++di) {
          if (d_ranks[b] == owner) continue;
          const int64_t lo = slo > d_ivs[2 * di] ? slo : d_ivs[2 * di];
          const int64_t hi = shi < d_ivs[2 * di + 1] ? shi : d_ivs[2 * di + 1];
          if (lo >= hi) continue;
          if (n >= cap) return -1;
          row5* r = (row5*)(out + 5 * n);
          r->src = phys;
          r->dst = d_ranks[b];
          r->lo = lo;
          r->hi = hi;
          r->medium = dead ? 1 : 0;
          ++n;
        }
      }
    }
  }
  qsort(out, (size_t)n, sizeof(row5), cmp_lo);
  return n;
}

/* ---------------- weighted reduce in fixed point ---------------- */

int ew_oracle_fixed_point_bits(double absmax, int64_t total_units) {
  if (absmax == 0.0) return 0;
  int e = 0;
  frexp(absmax, &e);
  int cu = 0;
  while (((int64_t)1 << cu) < total_units) ++cu;
  int f = 62 - e - cu;
  return f > 1000 ? 1000 : f;
}

/* acc[i] = sum_u rint_half_even(w_u * (double)g_u[i] * 2^F) */
void ew_oracle_weighted_fixed(const double* w, const float* g, int n_units, int64_t dim,
                              int frac_bits, int64_t* acc) {
  const double scale = ldexp(1.0, frac_bits);
  for (int64_t i = 0; i < dim; ++i) {
    int64_t s = 0;
    for (int u = 0; u < n_units; ++u) {
      const double prod = w[u] * (double)g[(int64_t)u * dim + i];
      s += (int64_t)nearbyint(prod * scale);
    }
    acc[i] = s;
  }
}

/* ---------------- multi-threaded CPU baseline (bench.py cpu_baseline) ----
 * Same definitions as above, organised for speed on host cores: each thread
 * takes whole checksum rows; a row whose global/local shift is a multiple of
 * 8 is checksummed word-wise (interior words straight from memory), other
 * rows fall back to the byte-serial definition.  Used only as the reported
 * CPU baseline ("port": the reference has no snapshot/checksum code). */
#include <pthread.h>

typedef struct {
  int64_t local_lo, len, delta, block;
} row_geom;

static int64_t build_rows(const int64_t* segs, int64_t n_segs, int64_t block, row_geom** out) {
  int64_t n = ew_oracle_num_rows(segs, n_segs, block), r = 0;
  row_geom* rows = (row_geom*)malloc(sizeof(row_geom) * (size_t)(n > 0 ? n : 1));
  for (int64_t k = 0; k < n_segs; ++k) {
    const int64_t glo = segs[3 * k], len = segs[3 * k + 1], loff = segs[3 * k + 2];
    if (len <= 0) continue;
    for (int64_t b = glo / block; b <= (glo + len - 1) / block; ++b, ++r) {
      const int64_t lo = glo > b * block ? glo : b * block;
      const int64_t hi = (glo + len) < (b + 1) * block ? (glo + len) : (b + 1) * block;
      rows[r].local_lo = lo - glo + loff;
      rows[r].len = hi - lo;
      rows[r].delta = glo - loff;
      rows[r].block = b;
    }
  }
  *out = rows;
  return n;
}

static void row_checksum(const row_geom* g, const uint8_t* buf, uint64_t* s0o, uint64_t* s1o) {
  const int64_t glo = g->local_lo + g->delta, ghi = glo + g->len;
  uint64_t s0 = 0, s1 = 0;
  int64_t i = glo / 8;
  const int64_t i_end = (ghi - 1) / 8;
  for (; i <= i_end; ++i) {
    uint64_t w = 0;
    if ((g->delta & 7) == 0 && 8 * i >= glo && 8 * i + 8 <= ghi) {
      memcpy(&w, buf + (8 * i - g->delta), 8);
    } else {
      for (int j = 0; j < 8; ++j) {
        const int64_t x = 8 * i + j;
        if (x >= glo && x < ghi) w |= (uint64_t)buf[x - g->delta] << (8 * j);
      }
    }
    s0 += w;
    s1 += (uint64_t)(i + 1) * w;
  }
  *s0o = s0;
  *s1o = s1;
}

typedef struct {
  const row_geom* rows;
  int64_t lo, hi;
  const uint8_t* src;
  uint8_t* dst;
  uint64_t* sums;
  const uint64_t* expected;
  int64_t bad;
} mt_job;

static void* mt_worker(void* p) {
  mt_job* j = (mt_job*)p;
  for (int64_t r = j->lo; r < j->hi; ++r) {
    const row_geom* g = &j->rows[r];
    if (j->dst) memcpy(j->dst + g->local_lo, j->src + g->local_lo, (size_t)g->len);
    uint64_t s0, s1;
    row_checksum(g, j->src, &s0, &s1);
    if (j->expected) {
      if (s0 != j->expected[2 * r] || s1 != j->expected[2 * r + 1]) ++j->bad;
    } else {
      j->sums[2 * r] = s0;
      j->sums[2 * r + 1] = s1;
    }
  }
  return NULL;
}

static int64_t run_mt(const int64_t* segs, int64_t n_segs, int64_t block, const uint8_t* src,
                      uint8_t* dst, uint64_t* sums, const uint64_t* expected, int threads) {
  row_geom* rows;
  const int64_t n = build_rows(segs, n_segs, block, &rows);
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  mt_job* jobs = (mt_job*)malloc(sizeof(mt_job) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (mt_job){rows, n * t / threads, n * (t + 1) / threads, src, dst, sums, expected, 0};
    pthread_create(&th[t], NULL, mt_worker, &jobs[t]);
  }
  int64_t bad = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    bad += jobs[t].bad;
  }
  free(th);
  free(jobs);
  free(rows);
  return bad;
}

/* snap <- live + row sums of live; returns 0 */
int64_t ew_oracle_snapshot_mt(const int64_t* segs, int64_t n_segs, int64_t block,
                              const uint8_t* live, uint8_t* snap, uint64_t* sums, int threads) {
  return run_mt(segs, n_segs, block, live, snap, sums, NULL, threads);
}

/* number of rows of buf whose sums differ from expected */
int64_t ew_oracle_verify_mt(const int64_t* segs, int64_t n_segs, int64_t block,
                            const uint8_t* buf, const uint64_t* expected, int threads) {
  return run_mt(segs, n_segs, block, buf, NULL, NULL, expected, threads);
}

/* ---- ring replica by optimizer replay -------------------
 * CPU restatement of ew_adam_step (include/ew_api.h): torch.optim.AdamW
 * (decoupled weight decay) with every operation an explicitly rounded fp32
 * op, fmaf where the device uses __fmaf_rn, scalars derived in fp64 and
 * rounded once.  Built with -ffp-contract=off so gcc adds no contraction.
 * The paper replays this step on the holder from the owner's gradient shard
 * (PAPER.md:363-372); the reference only models its time (param_fabric.hpp:
 * 86-96), so parity is pinned against torch.optim.AdamW in the tests. */
uint16_t ew_oracle_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FC0u;
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

void ew_oracle_adam_scalars(double lr, double b1, double b2, double eps, double wd, int64_t step,
                            float out8[8]) {
  const double bc1 = 1.0 - pow(b1, (double)step);
  const double bc2 = 1.0 - pow(b2, (double)step);
  out8[0] = (float)b1;
  out8[1] = (float)(1.0 - b1);
  out8[2] = (float)b2;
  out8[3] = (float)(1.0 - b2);
  out8[4] = (float)eps;
  out8[5] = (float)(lr / bc1);
  out8[6] = (float)(1.0 / sqrt(bc2));
  out8[7] = (float)(1.0 - lr * wd);
}

void ew_oracle_adam_step(const float* grad, float* master, float* exp_avg, float* exp_avg_sq,
                         uint16_t* param, int64_t n, double lr, double b1, double b2, double eps,
                         double wd, int64_t step) {
  float s[8];
  ew_oracle_adam_scalars(lr, b1, b2, eps, wd, step, s);
  for (int64_t i = 0; i < n; ++i) {
    const float g = grad[i];
    const float m1 = fmaf(s[0], exp_avg[i], s[1] * g);
    const float v1 = fmaf(s[2], exp_avg_sq[i], (s[3] * g) * g);
    const float denom = sqrtf(v1) * s[6] + s[4];
    const float p1 = fmaf(-s[5], m1 / denom, master[i] * s[7]);
    master[i] = p1;
    exp_avg[i] = m1;
    exp_avg_sq[i] = v1;
    param[i] = ew_oracle_bf16(p1);
  }
}

/* ---- multi-threaded CPU paths timed beside the GPU kernels (BASELINE §3) --
 * Reported baselines, not optimisation targets: the reference's own
 * functions are single-threaded planners/models, so these restate the byte
 * work on T host threads with the same per-element arithmetic. */
typedef struct {
  int64_t lo, hi;
  const uint8_t* const* src;
  uint8_t* const* dst;
  const int64_t* bytes;
  /* draw */
  uint64_t seed, sample_lo;
  uint32_t layer, op;
  int64_t n_per_sample;
  double* out;
  /* weighted average */
  const double* w;
  const double* g;
  int n_units;
  int64_t dim;
} cpu_job;

static void* copy_worker(void* p) {
  cpu_job* j = (cpu_job*)p;
  for (int64_t k = j->lo; k < j->hi; ++k) memcpy(j->dst[k], j->src[k], (size_t)j->bytes[k]);
  return NULL;
}

/* (b) plan execution: one memcpy per TransferEntry, entries split over T
 * threads (SURVEY §8(d) "builder CPU plan executor") */
void ew_oracle_memcpy_mt(const uint8_t* const* src, uint8_t* const* dst, const int64_t* bytes,
                         int64_t n, int threads) {
  if (threads < 1) threads = 1;
  pthread_t th[256];
  cpu_job jobs[256];
  if (threads > 256) threads = 256;
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (cpu_job){0};
    jobs[t].lo = n * t / threads;
    jobs[t].hi = n * (t + 1) / threads;
    jobs[t].src = src;
    jobs[t].dst = dst;
    jobs[t].bytes = bytes;
    pthread_create(&th[t], NULL, copy_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

static void* draw_worker(void* p) {
  cpu_job* j = (cpu_job*)p;
  for (int64_t s = j->lo; s < j->hi; ++s)
    ew_oracle_draw(j->seed, j->sample_lo + (uint64_t)s, j->layer, j->op, j->n_per_sample,
                   j->out + s * j->n_per_sample);
  return NULL;
}

/* (c) draw() (rng.cpp:38-53) over disjoint samples on T threads */
void ew_oracle_draw_mt(uint64_t seed, uint64_t sample_lo, int64_t n_samples, uint32_t layer,
                       uint32_t op, int64_t n_per_sample, double* out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  cpu_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (cpu_job){0};
    jobs[t].lo = n_samples * t / threads;
    jobs[t].hi = n_samples * (t + 1) / threads;
    jobs[t].seed = seed;
    jobs[t].sample_lo = sample_lo;
    jobs[t].layer = layer;
    jobs[t].op = op;
    jobs[t].n_per_sample = n_per_sample;
    jobs[t].out = out;
    pthread_create(&th[t], NULL, draw_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

static void* wavg_worker(void* p) {
  cpu_job* j = (cpu_job*)p;
  for (int64_t i = j->lo; i < j->hi; ++i) {
    double acc = 0.0;
    for (int u = 0; u < j->n_units; ++u) acc += j->w[u] * j->g[(int64_t)u * j->dim + i];
    j->out[i] = acc;
  }
  return NULL;
}

/* (d) weighted_grad_average (dataflow.cpp:71-83) element-parallel on T
 * threads with the reference's per-element left-fold order (bit-identical) */
void ew_oracle_weighted_average_mt(const double* w, const double* g, int n_units, int64_t dim,
                                   double* out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  cpu_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (cpu_job){0};
    jobs[t].lo = dim * t / threads;
    jobs[t].hi = dim * (t + 1) / threads;
    jobs[t].w = w;
    jobs[t].g = g;
    jobs[t].n_units = n_units;
    jobs[t].dim = dim;
    jobs[t].out = out;
    pthread_create(&th[t], NULL, wavg_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------------
 * Synthetic-state checksums without a buffer, on T threads (checker for
 * full-size GPU runs: config B rank shards of 11.8 GB, the 94.3 GB space).
 * A row / block is summed straight from w_i = splitmix64(seed ^ i), the
 * words at a range's ends masked to the bytes inside it. */
typedef struct {
  uint64_t seed;
  const row_geom* rows;
  int64_t lo, hi, block, total;
  uint64_t* out;
} synth_job;

static void range_sums_synthetic(uint64_t seed, int64_t glo, int64_t ghi, uint64_t* s0o,
                                 uint64_t* s1o) {
  uint64_t s0 = 0, s1 = 0;
  for (int64_t i = glo / 8; i <= (ghi - 1) / 8; ++i) {
    uint64_t w = ew_oracle_splitmix64(seed ^ (uint64_t)i);
    const int64_t a = glo > 8 * i ? glo - 8 * i : 0;        /* first byte kept */
    const int64_t e = ghi < 8 * i + 8 ? ghi - 8 * i : 8;    /* one past last   */
    if (a > 0) w &= ~0ULL << (8 * a);
    if (e < 8) w &= (1ULL << (8 * e)) - 1;
    s0 += w;
    s1 += (uint64_t)(i + 1) * w;
  }
  *s0o = s0;
  *s1o = s1;
}

static void* synth_rows_worker(void* p) {
  synth_job* j = (synth_job*)p;
  for (int64_t r = j->lo; r < j->hi; ++r) {
    const int64_t glo = j->rows[r].local_lo + j->rows[r].delta;
    range_sums_synthetic(j->seed, glo, glo + j->rows[r].len, &j->out[2 * r], &j->out[2 * r + 1]);
  }
  return NULL;
}

static void* synth_blocks_worker(void* p) {
  synth_job* j = (synth_job*)p;
  for (int64_t b = j->lo; b < j->hi; ++b) {
    const int64_t lo = b * j->block;
    const int64_t hi = lo + j->block < j->total ? lo + j->block : j->total;
    range_sums_synthetic(j->seed, lo, hi, &j->out[2 * b], &j->out[2 * b + 1]);
  }
  return NULL;
}

static void run_synth(void* (*fn)(void*), synth_job base, int64_t n, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  synth_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = base;
    jobs[t].lo = n * t / threads;
    jobs[t].hi = n * (t + 1) / threads;
    pthread_create(&th[t], NULL, fn, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* Rows (segment order, blocks ascending) of the synthetic state placed by
 * segs; returns the row count. */
int64_t ew_oracle_rows_synthetic_mt(uint64_t seed, const int64_t* segs, int64_t n_segs,
                                    int64_t block, uint64_t* out, int threads) {
  row_geom* rows = NULL;
  const int64_t n = build_rows(segs, n_segs, block, &rows);
  synth_job base = {seed, rows, 0, 0, block, 0, out};
  run_synth(synth_rows_worker, base, n, threads);
  free(rows);
  return n;
}

void ew_oracle_block_sums_synthetic_mt(uint64_t seed, int64_t total_bytes, int64_t block,
                                       uint64_t* out, int threads) {
  synth_job base = {seed, NULL, 0, 0, block, total_bytes, out};
  run_synth(synth_blocks_worker, base, (total_bytes + block - 1) / block, threads);
}

/* ew_oracle_fill_synthetic on T threads: the packed buffer [0, total) is cut
 * into T byte ranges, each thread fills the segment bytes inside its range. */
typedef struct {
  const int64_t* segs;
  int64_t n_segs, lo, hi;
  uint64_t seed;
  uint8_t* buf;
} fill_job;

static void* fill_worker(void* p) {
  fill_job* j = (fill_job*)p;
  for (int64_t k = 0; k < j->n_segs; ++k) {
    const int64_t glo = j->segs[3 * k], len = j->segs[3 * k + 1], loff = j->segs[3 * k + 2];
    const int64_t a = loff > j->lo ? loff : j->lo;
    const int64_t e = loff + len < j->hi ? loff + len : j->hi;
    for (int64_t x = a; x < e; ++x) {
      const int64_t g = glo + (x - loff);
      j->buf[x] = (uint8_t)(ew_oracle_splitmix64(j->seed ^ (uint64_t)(g / 8)) >> (8 * (g % 8)));
    }
  }
  return NULL;
}

void ew_oracle_fill_synthetic_mt(const int64_t* segs, int64_t n_segs, uint64_t seed,
                                 uint8_t* buf, int64_t total, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  fill_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (fill_job){segs, n_segs, total * t / threads, total * (t + 1) / threads, seed, buf};
    pthread_create(&th[t], NULL, fill_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}
