/* ew_api.h — C ABI of libelaskit_b200.so, the B200 build of ElasWave's
 * per-step data-parallel recovery path.
 *
 * The reference (proj/include/elaskit) is a C++ library with no FFI layer;
 * its C++ headers stay the primary API (the include/elaskit headers, implemented in
 * the same .so).  This header is what a foreign caller (ctypes, cgo, JNI) or
 * a C++ executor binds: plain pointers and sizes, integer status codes, no
 * exceptions and no torch types.  Each planning entry point names the
 * reference function it wraps; the device entry points execute what the
 * reference only models (SURVEY §2 "Modelled transfer" table).
 *
 * Conventions
 *   - Every function returns EW_OK (0) or an ew_status; ew_last_error() gives
 *     the message.  Status codes map 1:1 onto the reference's exception types
 *     (elaskit/device.hpp rethrows them).
 *   - Device pointers are caller-owned and live on the CUDA device current on
 *     the calling thread.  ew_stream_t is a cudaStream_t (NULL = default).
 *   - Device calls are asynchronous on the given stream unless stated.
 *   - Access granularity: the streaming kernels move memory with bulk (TMA)
 *     transfers that cover whole aligned granules — 16 bytes for copy
 *     sources (ew_copy_program_*), 32 bytes for snapshot / checksum / verify
 *     buffers.  A granule holding at least one byte of a caller's range may
 *     be read in full, so up to 15 (31) bytes before or past the range are
 *     READ (never written) and their values ignored.  Such a granule never
 *     straddles a 4 KiB page, so the over-read cannot fault on any mapping
 *     the range itself lives in (device allocations, IPC mappings,
 *     page-granular host registrations); callers need no padding.  Writes
 *     are byte-exact.
 */
#ifndef EW_API_H
#define EW_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ew_stream_t;

enum ew_status {
  EW_OK = 0,
  EW_ERR_INVALID_ARGUMENT = 1,   /* std::invalid_argument            */
  EW_ERR_COVERAGE_MISMATCH = 2,  /* elaskit::CoverageMismatch        */
  EW_ERR_MISSING_BACKUP = 3,     /* elaskit::MissingBackup           */
  EW_ERR_NO_SURVIVORS = 4,       /* elaskit::NoSurvivors             */
  EW_ERR_DIMENSION_MISMATCH = 5, /* elaskit::DimensionMismatch       */
  EW_ERR_MISMATCHED_DP = 6,      /* elaskit::MismatchedDpDegree      */
  EW_ERR_DISCONNECTED = 7,       /* elaskit::DisconnectedGroup       */
  EW_ERR_OUT_OF_RANGE = 8,       /* std::out_of_range                */
  EW_ERR_CAPACITY = 9,           /* output buffer too small          */
  EW_ERR_CUDA = 10,
  EW_ERR_NCCL = 11,
  EW_ERR_INTERNAL = 12,
  EW_ERR_INSUFFICIENT_MEMORY = 13 /* elaskit::InsufficientTargetMemory */
};

const char* ew_last_error(void);
const char* ew_version(void);

/* ------------------------------------------------------------------------
 * Layouts — PartitionLayout (reference param_fabric.hpp:27-33)
 * ---------------------------------------------------------------------- */
typedef struct ew_layout ew_layout;

typedef struct ew_interval {
  int64_t lo, hi; /* half-open */
} ew_interval;

/* One interval of a rank's packed shard buffer (elaskit/b200.hpp Segment). */
typedef struct ew_segment {
  int64_t global_lo, length, local_off;
} ew_segment;

/* Interleaved ZeRO over `ranks` (ZeroLayout::shard, migration.cpp:73-77,
 * composed per SURVEY §8(a) A4). */
int ew_layout_interleaved(const int64_t* layer_bytes, int n_layers, const int* ranks,
                          int n_ranks, ew_layout** out);
/* contiguous_layout (param_fabric.cpp:36-49) */
int ew_layout_contiguous(const int* ranks, int n_ranks, int64_t total, ew_layout** out);
/* Arbitrary layout: rank ranks[i] gets counts[i] consecutive entries of ivs. */
int ew_layout_from_intervals(const int* ranks, const int* counts, int n_ranks,
                             const ew_interval* ivs, int64_t total, ew_layout** out);
void ew_layout_free(ew_layout* layout);
int64_t ew_layout_total_bytes(const ew_layout* layout);
int ew_layout_num_ranks(const ew_layout* layout);
int ew_layout_ranks(const ew_layout* layout, int* out, int cap);
int64_t ew_layout_shard_bytes(const ew_layout* layout, int rank);
int64_t ew_layout_num_segments(const ew_layout* layout, int rank);
int ew_layout_segments(const ew_layout* layout, int rank, ew_segment* out, int64_t cap);
/* PartitionLayout::validate (param_fabric.cpp:14-34) */
int ew_layout_validate(const ew_layout* layout);
/* PartitionLayout::owner_of (param_fabric.cpp:7-12); -1 if uncovered */
int ew_layout_owner_of(const ew_layout* layout, int64_t byte);

/* integrity_check (param_fabric.cpp:66-80).  *recoverable = 0/1; the failed
 * ranks whose holder also failed are written to missing_ranks. */
int ew_integrity_check(const int* ring_members, int n_ring, const ew_layout* layout,
                       const int* failed, int n_failed, int* recoverable, int* missing_ranks,
                       int missing_cap, int* n_missing);

/* ------------------------------------------------------------------------
 * Transfer plans — overlap_matrix (param_fabric.cpp:82-121)
 * ---------------------------------------------------------------------- */
typedef struct ew_plan ew_plan;

enum { EW_MEDIUM_D2D = 0, EW_MEDIUM_H2D_D2D = 1 };

typedef struct ew_transfer_entry {
  int32_t src_rank, dst_rank;
  int64_t lo, hi;
  int32_t medium, reserved;
} ew_transfer_entry;

/* n_ring == 0 passes ring = nullptr, like the reference default argument. */
int ew_overlap_matrix(const ew_layout* src, const ew_layout* dst, const int* failed,
                      int n_failed, const int* ring_members, int n_ring, ew_plan** out);
void ew_plan_free(ew_plan* plan);
int64_t ew_plan_num_entries(const ew_plan* plan);
int64_t ew_plan_total_bytes_moved(const ew_plan* plan);
int ew_plan_entries(const ew_plan* plan, ew_transfer_entry* out, int64_t cap);
/* plan_to_json (param_fabric.cpp:123-134), compact dump, NUL-terminated. */
int ew_plan_to_json(const ew_plan* plan, char* buf, int64_t cap, int64_t* needed);

enum { EW_ROLE_OLD = 0, EW_ROLE_REPLICA = 1, EW_ROLE_NEW = 2 };

typedef struct ew_copy_desc {
  int32_t src_role, src_rank, dst_role, dst_rank;
  int64_t src_off, dst_off, bytes;
} ew_copy_desc;

/* Lower a plan to the copies GPU `exec_rank` issues (b200.hpp reshard_copies).
 * push != 0: copies sourced on exec_rank; push == 0: copies landing there.
 * Writes min(n, cap) descriptors and *n_out = n (EW_ERR_CAPACITY if n > cap). */
int ew_reshard_copies(const ew_plan* plan, const ew_layout* src, const ew_layout* dst,
                      const int* failed, int n_failed, const int* ring_members, int n_ring,
                      int exec_rank, int push, ew_copy_desc* out, int64_t cap, int64_t* n_out);

/* Staged in-place reshard schedule (b200.hpp inplace_schedule; config D):
 * OLD and NEW share one buffer per rank, the plan's copies run in phases.
 * Phases are global [lo, hi) pairs in processing order; per rank and phase,
 * `cut` is the packed NEW range, `direct` the part gather_j writes in place,
 * `staged` the part it stages and flushes after the phase's barrier.
 * Ranges of a rank are arrays of 2 * n_phases int64.  ew_inplace_schedule
 * fails with EW_ERR_INVALID_ARGUMENT when shards neither all grow nor all
 * shrink, EW_ERR_COVERAGE_MISMATCH if the hazard check fails. */
typedef struct ew_inplace ew_inplace;
int ew_inplace_schedule(const int64_t* layer_bytes, int n_layers, const ew_layout* src,
                        const ew_layout* dst, const int* failed, int n_failed,
                        int64_t stage_bytes, int64_t phase_bytes, int slack, ew_inplace** out);
int ew_inplace_info(const ew_inplace* s, int* descending, int* slack, int* ring,
                    int64_t* n_phases, int64_t* stage_alloc);
int ew_inplace_phases(const ew_inplace* s, int64_t* out);
int ew_inplace_ranges(const ew_inplace* s, int rank, int64_t* cut, int64_t* direct,
                      int64_t* staged);
void ew_inplace_free(ew_inplace* s);

/* ------------------------------------------------------------------------
 * Host planners of the other hot-path modules
 * ---------------------------------------------------------------------- */
/* reshard_microbatches (dataflow.cpp:52-69): out arrays hold n_survivors. */
int ew_reshard_microbatches(const int* old_per_slot_mbs, int n_old, int num_microbatches,
                            const int* survivors, int n_survivors, int* out_slots,
                            int* out_per_slot_mbs);
/* SampleReassignment derivation of recover_elaswave (sim.cpp:694-715) between
 * two assignments: rows {sample_offset, old_slot, new_slot}. */
int ew_sample_reassignments(const int* old_slots, const int* old_mbs, int n_old,
                            const int* new_slots, const int* new_mbs, int n_new, int64_t* rows,
                            int64_t cap, int64_t* n_out);
/* plan_zero_migration (migration.cpp:87-154): kind 0 = Contiguous,
 * 1 = Interleaved; rows {src, dst, cross_stage, lo, hi, round};
 * totals {cross, intra, total}. */
int ew_plan_zero_migration(int kind, int dp_degree, const int64_t* layer_bytes, int n_layers,
                           int layer_idx, int dst_dp_degree, int64_t* rows, int64_t cap,
                           int64_t* n_out, int64_t* totals);
/* plan_layer_migration (migration.cpp:9-61): mode 0 = Blocking,
 * 1 = NonBlocking.  Fields mirror MigrationContext / MigrationSchedule
 * (migration.hpp:22-46); transfers[k].what: 0 = "params", 1 = "payback_grad". */
typedef struct ew_migration_context {
  int64_t param_bytes, grad_bytes;
  double link_bw_bytes_per_s, microbatch_slot_s;
  int32_t num_microbatches;
  int64_t target_headroom_bytes;
  double fixed_overhead_s;
} ew_migration_context;
typedef struct ew_transfer_segment {
  int32_t what;
  double start_s, end_s;
  int64_t bytes;
} ew_transfer_segment;
typedef struct ew_migration_schedule {
  int32_t mode, shadow_microbatches, n_transfers;
  ew_transfer_segment transfers[2];
  int64_t payback_bytes;
  double stall_s, total_time_s;
} ew_migration_schedule;
int ew_plan_layer_migration(int layer, int src_stage, int dst_stage, int mode,
                            const ew_migration_context* ctx, ew_migration_schedule* out);
/* weighted_grad_average (dataflow.cpp:71-83), fp64, grads row-major [n][dim] */
int ew_weighted_grad_average(const double* weights, const double* grads, int n, int64_t dim,
                             double* out);
/* philox4x64 (rng.cpp:25-36) and draw (rng.cpp:38-53) */
int ew_philox4x64(const uint64_t counter[4], const uint64_t key[2], uint64_t out[4]);
int ew_draw(uint64_t seed, uint64_t sample_id, uint32_t layer_id, uint32_t op_index, int n,
            double* out);

/* plan_edit (communicator.cpp:54-105).  Groups are given as flat member
 * lists; topo[i] 0 = Mesh, 1 = Ring; ids are NUL-terminated strings.  Links
 * are (lo,hi) pairs.  Outputs are truncated at their caps (EW_ERR_CAPACITY). */
int ew_plan_edit(int n_groups, const char* const* ids, const int* topo, const int* n_members,
                 const int* members, int event_kind, const int* targets, int n_targets,
                 const int* pool_links, int n_pool, int* add_links, int add_cap, int* n_add,
                 int* remove_links, int remove_cap, int* n_remove, int* touched_groups,
                 int* n_touched);

/* ------------------------------------------------------------------------
 * Device memory and peer mappings (B200 "links": CUDA IPC over NVSwitch)
 * ---------------------------------------------------------------------- */
int ew_device_count(int* n);
int ew_set_device(int device);
/* Map peer_device's memory into the current device's address space (one
 * process driving several GPUs; processes use CUDA IPC instead). */
int ew_peer_access_enable(int peer_device);
int ew_alloc(int64_t bytes, void** out); /* cudaMalloc, 256-B aligned, current device */
int ew_free(void* ptr);
int ew_memset_async(void* ptr, int value, int64_t bytes, ew_stream_t stream);
int ew_memcpy_async(void* dst, const void* src, int64_t bytes, ew_stream_t stream);
int ew_stream_sync(ew_stream_t stream);
int ew_device_sync(void);
/* 64-byte cudaIpcMemHandle of the allocation holding ptr + ptr's offset. */
int ew_ipc_get_handle(const void* ptr, void* handle64, int64_t* offset);
int ew_ipc_open(const void* handle64, int64_t offset, void** out);
int ew_ipc_close(void* ptr);
/* Host memory as a transfer source (Medium::H2D_D2D, param_fabric.hpp:63):
 * pin [host, host + bytes) for every device of this process (portable,
 * mapped) and return the device address the copy kernels read it through
 * over PCIe.  `host` may be node-shared memory (POSIX shm) that other ranks
 * register too.  Unregister before unmapping the range. */
int ew_host_register(void* host, int64_t bytes, void** dev_ptr);
int ew_host_unregister(void* host);
/* Stream-ordered store of one u64 (a commit word), e.g. into registered host
 * memory through its device address, after the stream's earlier copies. */
int ew_write_u64_async(void* dev_ptr, uint64_t value, ew_stream_t stream);

/* ------------------------------------------------------------------------
 * (a) Snapshot + per-block checksum, verification
 *
 * Checksum spec (builder-defined; the reference has none — parity unpinned,
 * see oracle/ew_oracle.c): the flat byte space is cut into blocks of
 * block_bytes (power of two, 4 KiB..1 MiB).  For global little-endian u64
 * word i (bytes [8i, 8i+8)) with the bytes a buffer does not hold read as 0,
 *     s0(b) = sum w_i,  s1(b) = sum (i+1) * w_i   (mod 2^64)
 * over the words of block b.  A "row" is (segment, block) and carries the
 * partial sums of the bytes of that segment inside that block; rows of all
 * ranks add up (mod 2^64) to the block sums of the whole space, for any
 * layout — reshard verification needs no re-read of the source.
 * ---------------------------------------------------------------------- */
typedef struct ew_shardmap ew_shardmap;

/* segs: ascending global order, local_off tiling [0, total) back to back.
 * The map keeps a device row table (32 B per row: e.g. 5.8 MB for a 7B rank
 * shard at 64 KiB blocks) for the snapshot / checksum / verify kernel. */
int ew_shardmap_create(const ew_segment* segs, int64_t n_segs, int64_t block_bytes,
                       ew_shardmap** out);
void ew_shardmap_free(ew_shardmap* map);
int64_t ew_shardmap_bytes(const ew_shardmap* map);
int64_t ew_shardmap_num_rows(const ew_shardmap* map);
int ew_shardmap_row_blocks(const ew_shardmap* map, int64_t* out_block_ids, int64_t cap);

/* snap <- live (whole packed buffer) fused with row checksums of live.
 * live/snap 32-byte aligned (256-bit accesses; ew_checksum / ew_verify
 * likewise); row_sums: device uint64[2 * num_rows]. */
int ew_snapshot(const ew_shardmap* map, const void* live, void* snap, uint64_t* row_sums,
                ew_stream_t stream);
int ew_checksum(const ew_shardmap* map, const void* buf, uint64_t* row_sums,
                ew_stream_t stream);
/* Recompute rows of buf and compare with expected.  *bad_count (device
 * uint32, zeroed by the call) receives the number of mismatching rows, whose
 * indices go to bad_rows[0..bad_cap) when bad_rows != NULL. */
int ew_verify(const ew_shardmap* map, const void* buf, const uint64_t* expected_row_sums,
              uint32_t* bad_count, int64_t* bad_rows, int64_t bad_cap, ew_stream_t stream);
/* block_sums[2*b .. 2*b+1] += row sums of the rows in global block b. */
int ew_rows_to_blocks(const ew_shardmap* map, const uint64_t* row_sums, uint64_t* block_sums,
                      int64_t n_blocks, ew_stream_t stream);
/* Synthetic model state: global word i = splitmix64(seed ^ i), placed by the
 * segment map (any rank can regenerate any interval). */
int ew_fill_synthetic(const ew_shardmap* map, void* buf, uint64_t seed, ew_stream_t stream);

/* ------------------------------------------------------------------------
 * (b) Reshard executor — peer-pointer copies over NVLink/NVSwitch
 * ---------------------------------------------------------------------- */
typedef struct ew_copy_program ew_copy_program;

/* Resolve descriptors against buf_table[role * table_ranks + rank] (local or
 * IPC-mapped peer pointers; NULL where absent) and upload the program to the
 * current device.  Copies whose destination is not on exec_rank are "remote". */
int ew_copy_program_create(const ew_copy_desc* descs, int64_t n, void* const* buf_table,
                           int table_ranks, int exec_rank, ew_copy_program** out);
/* Program from already-resolved pointers (src, dst, bytes, is_remote). */
int ew_copy_program_create_raw(const void* const* srcs, void* const* dsts, const int64_t* bytes,
                               const int* is_remote, int64_t n, ew_copy_program** out);
void ew_copy_program_free(ew_copy_program* prog);
int ew_copy_program_stats(const ew_copy_program* prog, int64_t* n_copies, int64_t* remote_bytes,
                          int64_t* local_bytes);
/* One launch: remote copies on the first CTAs, local copies on the rest.
 * n_ctas == 0 picks 2 CTAs per SM; remote_ctas == 0 (or out of range) gives
 * the remote class a quarter of them when the program has both classes. */
int ew_copy_program_launch(const ew_copy_program* prog, int n_ctas, int remote_ctas,
                           ew_stream_t stream);
/* Same launch, gated on a device flag (e.g. ew_peer_barrier_error_flag): if
 * *abort_flag != 0 when the kernel starts, it writes nothing.  block_sums may
 * be NULL (plain program) or the verified program's block sums. */
int ew_copy_program_launch_guarded(const ew_copy_program* prog, int n_ctas, int remote_ctas,
                                   uint64_t* block_sums, const int* abort_flag,
                                   ew_stream_t stream);
/* Verification on arrival.  A verified program also checksums (kernel (a)'s
 * spec) every byte it lands in this GPU's NEW buffer, labelled with the
 * global position that byte's destination offset has in new_map (NEW's
 * segment map on exec_rank), and adds the sums into block_sums (device
 * u64 [n_blocks][2], caller-zeroed; n_blocks from ew_copy_program_num_blocks
 * covers global blocks up to NEW's last byte).  In-place retained bytes are
 * read and checksummed but not rewritten.  When every byte landed where the
 * target layout says, the sum of every NEW rank's block_sums equals the block
 * sums of the source state, with no re-read of NEW.  The converse is
 * probabilistic: the checksum is linear mod 2^64, so a misplaced or corrupted
 * landing goes unnoticed only if its error terms cancel in both s0 and s1 of
 * every block (a swap of two equal words, or a crafted collision). */
int ew_copy_program_create_verified(const ew_copy_desc* descs, int64_t n,
                                    void* const* buf_table, int table_ranks, int exec_rank,
                                    const ew_shardmap* new_map, ew_copy_program** out);
int ew_copy_program_launch_verified(const ew_copy_program* prog, int n_ctas, int remote_ctas,
                                    uint64_t* block_sums, ew_stream_t stream);
int ew_copy_program_num_blocks(const ew_copy_program* prog, int64_t* n_blocks);

/* ------------------------------------------------------------------------
 * (c) Philox-4x64-10 dropout masks keyed by global sample id
 * ---------------------------------------------------------------------- */
/* bits[s][k/32] bit (k%32) = 1 iff element k of sample sample_lo+s is KEPT
 * (reference rule sim.cpp:926-928: dropped iff u < keep_probability); rows
 * are ceil(n_elems/32) words, trailing bits 0. */
int ew_philox_dropout_mask(uint64_t seed, uint64_t sample_lo, int64_t n_samples,
                           uint32_t layer_id, uint32_t op_index, int64_t n_elems,
                           double keep_probability, uint32_t* bits, ew_stream_t stream);
/* out[s][k] = draw({seed, sample_lo+s, layer, op}, n_elems)[k].  Sample ids
 * are the reference's uint64 RngKey::sample_id (rng.hpp:21-26) over the full
 * domain; sample_lo + s wraps mod 2^64 as the reference's does. */
int ew_philox_uniforms(uint64_t seed, uint64_t sample_lo, int64_t n_samples, uint32_t layer_id,
                       uint32_t op_index, int64_t n_elems, double* out, ew_stream_t stream);
/* raw words of blocks block_lo .. block_lo+n_blocks-1 of one stream */
int ew_philox_words(uint64_t seed, uint64_t sample_id, uint32_t layer_id, uint32_t op_index,
                    uint64_t block_lo, int64_t n_blocks, uint64_t* out, ew_stream_t stream);

/* ------------------------------------------------------------------------
 * (d) Gradient-scale-preserving weighted reduce
 *
 * Each contribution unit u (a micro-batch or per-sample gradient, fp32 on
 * device) is scaled by its weight in fp64 and rounded to int64 fixed point
 * with frac_bits fractional bits; integer sums are exact and associative, so
 * the result does not depend on how units are split across ranks.
 * ---------------------------------------------------------------------- */
/* max_u,i |w_u * g_u[i]| into *out_max (device double; written, not max-ed). */
int ew_weighted_absmax(const float* const* units, const double* weights, int n_units,
                       int64_t n_elems, double* out_max, ew_stream_t stream);
/* Largest frac_bits with total_units * absmax * 2^frac_bits < 2^62. */
int ew_fixed_point_bits(double global_absmax, int64_t total_units, int* frac_bits);
/* acc[i] (+)= sum_u rint(w_u * g_u[i] * 2^frac_bits) */
int ew_weighted_fold(const float* const* units, const double* weights, int n_units,
                     int64_t n_elems, int frac_bits, int64_t* acc, int accumulate,
                     ew_stream_t stream);
/* The same steps with the scale in device memory (no host round trip: the
 * whole (d) step is stream-ordered and CUDA-graph capturable).
 * ew_fixed_point_bits_async writes ew_fixed_point_bits(*global_absmax,
 * total_units) to *frac_bits (device int), INT_MIN for a non-finite or
 * negative absmax (the _dev fold and dequant then produce zeros; check the
 * bits after the step). */
int ew_fixed_point_bits_async(const double* global_absmax, int64_t total_units, int* frac_bits,
                              ew_stream_t stream);
int ew_weighted_fold_dev(const float* const* units, const double* weights, int n_units,
                         int64_t n_elems, const int* frac_bits, int64_t* acc, int accumulate,
                         const int64_t* addend, ew_stream_t stream);
int ew_fixed_to_float_dev(const int64_t* acc, int64_t n, const int* frac_bits, float* out,
                          ew_stream_t stream);
/* Shadow-gradient payback of a non-blocking layer migration: acc[i] +=
 * payback[i] (int64 fixed point, so the split of micro-batches between the
 * source's shadow instance and the target is bit-exactly invisible).
 * payback may be a peer (IPC) pointer: the pull and the add are one pass. */
int ew_payback_accumulate(int64_t* acc, const int64_t* payback, int64_t n, ew_stream_t stream);
/* Same, plus acc[i] += addend[i] in the same pass (addend: int64, device or
 * peer pointer; NULL = none) — used to fold a migration's payback into the
 * target's last micro-batch instead of a separate pass. */
int ew_weighted_fold_addend(const float* const* units, const double* weights, int n_units,
                            int64_t n_elems, int frac_bits, int64_t* acc, int accumulate,
                            const int64_t* addend, ew_stream_t stream);
int ew_fixed_to_float(const int64_t* acc, int64_t n, int frac_bits, float* out,
                      ew_stream_t stream);
int ew_fixed_to_double(const int64_t* acc, int64_t n, int frac_bits, double* out,
                       ew_stream_t stream);

/* NCCL communicator of the DP group (the B200 "dynamic communicator"). */
typedef struct ew_comm ew_comm;
int ew_comm_unique_id(void* id128);
int ew_comm_init(const void* id128, int nranks, int rank, ew_comm** out);
/* ncclCommShrink: every non-excluded rank calls this; abort != 0 uses
 * NCCL_SHRINK_ABORT (a member died mid-operation). */
int ew_comm_shrink(ew_comm* parent, const int* exclude_ranks, int n_exclude, int abort,
                   ew_comm** out);
/* ncclCommSplit: every rank of `parent` calls it; color < 0 (NCCL_SPLIT_NOCOLOR)
 * leaves this rank out (*out = NULL).  share != 0 shares the parent's
 * buffers and connections (splitShare): a split prepared in steady state for
 * every possible departure then costs little memory, and the repair at
 * failure time is a lookup (recovery.hpp DpGroup). */
int ew_comm_split(ew_comm* parent, int color, int key, int share, ew_comm** out);
int ew_comm_rank(const ew_comm* comm, int* rank, int* nranks);
/* ncclCommAbort: frees the communicator without waiting for its peers (a
 * communicator that includes a departed rank; ncclCommDestroy may block on
 * peers that will never arrive). */
int ew_comm_abort(ew_comm* comm);
int ew_comm_destroy(ew_comm* comm);
/* In-place sums over the communicator. */
int ew_allreduce_i64(ew_comm* comm, int64_t* buf, int64_t n, ew_stream_t stream);
int ew_allreduce_u64(ew_comm* comm, uint64_t* buf, int64_t n, ew_stream_t stream);
int ew_allreduce_max_f64(ew_comm* comm, double* buf, int64_t n, ew_stream_t stream);
/* Full (d): absmax pre-pass -> NCCL max -> fold -> NCCL int64 sum -> fp32.
 * total_units is the global unit count; ws_acc holds n_elems int64,
 * ws_max one double; *frac_bits_out (host) receives the scale used.  This
 * call synchronises the stream once to read the global max. */
int ew_weighted_reduce(ew_comm* comm, const float* const* units, const double* weights,
                       int n_units, int64_t total_units, int64_t n_elems, int64_t* ws_acc,
                       double* ws_max, float* out, int* frac_bits_out, ew_stream_t stream);
/* Same, fully asynchronous: the scale lives in *ws_bits (device int); no host
 * synchronisation, so the step can be captured in a CUDA graph. */
int ew_weighted_reduce_async(ew_comm* comm, const float* const* units, const double* weights,
                             int n_units, int64_t total_units, int64_t n_elems, int64_t* ws_acc,
                             double* ws_max, int* ws_bits, float* out, ew_stream_t stream);

/* (d) fused with its collective over NVLink peer memory (no NCCL): the same
 * quantised int64 sums, bit-identical to ew_weighted_reduce.  unit_ptrs lists
 * EVERY rank's units (IPC-mapped peer pointers or local ones), out_ptrs every
 * rank's fp32 output buffer; all 16-byte aligned.  Call reduce_scatter on all
 * ranks, make sure every rank finished it (a host barrier), then all_gather;
 * the caller also barriers before the units are read. */
typedef struct ew_peer_fold ew_peer_fold;
int ew_peer_fold_create(int world, int rank, int64_t n_elems, const float* const* unit_ptrs,
                        const double* unit_weights, int n_units, float* const* out_ptrs,
                        ew_peer_fold** out);
/* Same collective over per-rank int64 accumulators (each rank folded its own
 * micro-batch units with ew_weighted_fold, accumulate=1): acc_ptrs lists every
 * rank's accumulator (IPC-mapped or local), 16-byte aligned.  Reduce-scatter
 * sums the int64 values exactly and dequantises with frac_bits. */
int ew_peer_fold_create_i64(int world, int rank, int64_t n_elems, const int64_t* const* acc_ptrs,
                            float* const* out_ptrs, ew_peer_fold** out);
int ew_peer_fold_reduce_scatter(ew_peer_fold* fold, int frac_bits, ew_stream_t stream);
int ew_peer_fold_all_gather(ew_peer_fold* fold, ew_stream_t stream);
void ew_peer_fold_free(ew_peer_fold* fold);

/* Checksum conservation over peer memory (reshard verification): counts the
 * words i in [lo, hi) (even bounds: whole blocks) where
 *   sum_k plus[k][i] != sum_k minus[k][i]   (mod 2^64)
 * with plus / minus local or IPC-mapped u64 arrays (16-byte aligned).  Each
 * survivor checks its slice; *bad_count (device u32) is zeroed by run(). */
typedef struct ew_block_verifier ew_block_verifier;
int ew_block_verifier_create(const uint64_t* const* plus, int n_plus, const uint64_t* const* minus,
                             int n_minus, int64_t lo, int64_t hi, ew_block_verifier** out);
int ew_block_verifier_run(const ew_block_verifier* v, uint32_t* bad_count, ew_stream_t stream);
void ew_block_verifier_free(ew_block_verifier* v);

/* Stream-ordered barrier across the GPUs of a group over peer memory.
 * flag_ptrs[r] is rank r's zero-initialised uint64[world] array (IPC-mapped
 * on the other ranks).  Every rank enqueues wait() the same number of times;
 * a rank that never arrives makes the others give up after timeout_s and
 * report it through timed_out() (no hang). */
typedef struct ew_peer_barrier ew_peer_barrier;
int ew_peer_barrier_create(int world, int rank, unsigned long long* const* flag_ptrs,
                           ew_peer_barrier** out);
int ew_peer_barrier_wait(ew_peer_barrier* barrier, double timeout_s, ew_stream_t stream);
int ew_peer_barrier_timed_out(ew_peer_barrier* barrier, int* timed_out);
/* Device int the barrier sets to 1 on a timeout (and never clears): pass it to
 * ew_copy_program_launch_guarded so writes ordered after a failed barrier do
 * not run (an in-place reshard must not overwrite OLD bytes a lagging peer
 * has not read yet). */
int ew_peer_barrier_error_flag(ew_peer_barrier* barrier, const int** flag);
void ew_peer_barrier_free(ew_peer_barrier* barrier);

/* ------------------------------------------------------------------------
 * Ring replica by optimizer replay: the
 * holder of member r's replica applies r's AdamW step from r's reduced
 * gradient shard (read over NVLink through an IPC pointer) instead of pulling
 * r's whole 14 B/param state.  The owner runs the same call as its own
 * optimizer step, so the replica stays byte-identical and r's checksum rows
 * verify it.  Per element (torch.optim.AdamW, every op IEEE-rounded, no
 * contraction):
 *   m' = fma(b1, m, (1-b1)*g)          v' = fma(b2, v, ((1-b2)*g)*g)
 *   d  = sqrt(v') * (1/sqrt(bc2)) + eps
 *   p' = fma(-lr/bc1, m'/d, p*(1-lr*wd))   param_bf16 = bf16_rne(p')
 * with bc_k = 1 - b_k^step and the scalars rounded to fp32 once on the host.
 * ---------------------------------------------------------------------- */
typedef struct ew_adam_hyper {
  double lr, beta1, beta2, eps, weight_decay;
} ew_adam_hyper;
/* out8 = {b1, 1-b1, b2, 1-b2, eps, lr/bc1, 1/sqrt(bc2), 1-lr*wd} as fp32 */
int ew_adam_scalars(const ew_adam_hyper* hyper, int64_t step, float* out8);
/* In place over n elements; grad may be a peer (IPC) pointer.  fp32 arrays
 * 16-byte aligned, param_bf16 8-byte aligned; step >= 1. */
int ew_adam_step(const float* grad, float* master, float* exp_avg, float* exp_avg_sq,
                 uint16_t* param_bf16, int64_t n, const ew_adam_hyper* hyper, int64_t step,
                 ew_stream_t stream);
/* Same step with kernel (a)'s checksum rows of the whole state image fused
 * in: the four arrays lie inside [image_base, image_base + image_bytes)
 * (bytes of the image the step does not write must be zero), rows
 * (device u64 [ceil(image_bytes/block_bytes)][2]) are overwritten with the
 * per-block (s0, s1) of the image after the step — equal to ew_checksum of
 * the image as one segment at global offset 0, without re-reading it. */
int ew_adam_step_rows(const float* grad, float* master, float* exp_avg, float* exp_avg_sq,
                      uint16_t* param_bf16, int64_t n, const ew_adam_hyper* hyper, int64_t step,
                      const void* image_base, int64_t image_bytes, int64_t block_bytes,
                      uint64_t* rows, ew_stream_t stream);
/* *bad_count (device u32, zeroed by the call) = rows where a != b. */
int ew_rows_diff(const uint64_t* a, const uint64_t* b, int64_t n_rows, uint32_t* bad_count,
                 ew_stream_t stream);

/* ------------------------------------------------------------------------
 * Multi-process recovery runtime (include/elaskit/recovery.hpp): the DP
 * slice of the reference's recover_elaswave (sim.cpp:597-722) executed
 * across processes — one per GPU, or several sharing one GPU.  Ranks meet
 * through a key-value store (plumbing only: IPC handles, barriers, verdict
 * counts); state and checksums move GPU to GPU through peer pointers.
 * ---------------------------------------------------------------------- */
typedef struct ew_store ew_store;
/* TCP store hosted by the is_server process on host:port (a listening
 * thread); every process, the host included, connects to it. */
int ew_store_tcp(const char* host, int port, int is_server, double timeout_s, ew_store** out);
/* Store over caller callbacks (e.g. torch.distributed's c10d store).  get
 * blocks until the key exists, writes min(len, cap) bytes and *len; it
 * returns EW_ERR_CAPACITY when cap < *len (the library retries once with a
 * buffer of *len bytes), another nonzero value on failure. */
typedef int (*ew_store_set_fn)(void* ctx, const char* key, int64_t key_len, const char* val,
                               int64_t len);
typedef int (*ew_store_get_fn)(void* ctx, const char* key, int64_t key_len, char* buf,
                               int64_t cap, int64_t* len);
/* erase (may be NULL): drop a key no member will read again; channels erase
 * their keys two rounds behind, so a store holds O(channels x members). */
typedef int (*ew_store_erase_fn)(void* ctx, const char* key, int64_t key_len);
int ew_store_callbacks(ew_store_set_fn set, ew_store_get_fn get, ew_store_erase_fn erase,
                       void* ctx, ew_store** out);
int ew_store_set(ew_store* store, const char* key, const void* val, int64_t len);
int ew_store_get(ew_store* store, const char* key, void* buf, int64_t cap, int64_t* len);
void ew_store_free(ew_store* store);

/* Ordered member list on a store; collectives name their keys by channel
 * name and call count, so every member makes the same sequence of calls. */
typedef struct ew_channel ew_channel;
int ew_channel_create(ew_store* store, const char* name, const int* members, int n, int me,
                      ew_channel** out);
int ew_channel_barrier(ew_channel* ch);
int ew_channel_sum(ew_channel* ch, int64_t mine, int64_t* total);
void ew_channel_free(ew_channel* ch);

/* MttrEvent (reference sim.hpp:31-45) with measured phases; phases a path
 * does not run read -1. */
typedef struct ew_mttr_event {
  int32_t step, verified;
  double t_event_s;
  char kind[16];
  double detect_s, comm_repair_s, remap_s, migration_stall_s, other_s, lost_work_s;
  double plan_edit_s, comm_acquire_s, first_collective_s, comm_prepared;
  double plan_s, map_bind_s, copy_s, barrier_verify_s, verdict_exchange_s, launch_to_verdict_s;
  double mismatched_block_words, barrier_timeouts;
  double premapped; /* 1: the event used the group's steady-state peer mapping */
  double sums_s, bind_s; /* map_bind_s split: source block sums; lowering + program build */
  double prepared; /* 1: the event launched a program prepared in steady state */
  double stale_snapshots; /* participants whose snapshot step differs from the event's */
} ew_mttr_event;
/* mttr.csv (reference sim.cpp:1119-1132): header line and one row, no '\n' */
int ew_mttr_csv_header(char* buf, int64_t cap);
int ew_mttr_csv_row(const ew_mttr_event* ev, int index, char* buf, int64_t cap);

/* Peer buffer table: (key, member) -> device pointer; keys 0/1/2 are the
 * OLD / REPLICA / NEW roles of ew_copy_desc.  exchange() is collective over
 * the channel: publishes this rank's (key, ptr) pairs as CUDA IPC handles and
 * maps every other member's. */
typedef struct ew_peers ew_peers;
int ew_peers_create(ew_peers** out);
int ew_peers_exchange(ew_peers* peers, ew_channel* ch, const int* keys, void* const* ptrs, int n);
int ew_peers_put(ew_peers* peers, int key, int member, void* ptr);
int ew_peers_get(const ew_peers* peers, int key, int member, void** ptr);
void ew_peers_free(ew_peers* peers);

/* One rank's reshard executor over arbitrary layouts (overlap_matrix +
 * reshard_copies); bind() resolves its copies against a peer table (own
 * buffers put in it too), verify != 0 (pull) checksums what lands. */
typedef struct ew_reshard ew_reshard;
int ew_reshard_create(const ew_layout* src, const ew_layout* dst, const int* failed, int n_failed,
                      const int* ring_members, int n_ring, int me, int push, int64_t block_bytes,
                      ew_reshard** out);
int ew_reshard_bind(ew_reshard* r, const ew_peers* peers, int verify);
int ew_reshard_launch(const ew_reshard* r, uint64_t* block_sums, const int* abort_flag,
                      int n_ctas, int remote_ctas, ew_stream_t stream);
void ew_reshard_free(ew_reshard* r);

/* Every single departure of an interleaved-ZeRO DP group planned, lowered
 * and bound in steady state (collective over the channel's members).
 * old_rows / replica_rows: the per-step snapshot's checksum rows of this
 * rank's OLD shard and of the replica it keeps (NULL: re-read here).
 * flags bit 0: replica-aware sourcing — copies the plan sources from the OLD
 * shard of the member this rank backs up read this rank's (current) replica
 * of it instead, in local HBM (b200::prefer_local_replica).
 * new_buf: caller-owned NEW buffer of new_capacity bytes, large enough for
 * every departure (NULL: allocated here).  recover() (survivors only, all of
 * them): one verified copy launch into the NEW buffer, a device barrier,
 * checksum conservation over peer memory, the verdict summed over the
 * survivors. */
typedef struct ew_prepared ew_prepared;
int ew_prepared_create(ew_channel* ch, const int64_t* layer_bytes, int n_layers, void* old_buf,
                       const uint64_t* old_rows, void* replica, const uint64_t* replica_rows,
                       void* new_buf, int64_t new_capacity, int64_t block_bytes,
                       double barrier_timeout_s, int flags, ew_prepared** out);
int ew_prepared_recover(ew_prepared* p, int departed, ew_stream_t stream, ew_mttr_event* ev,
                        int* verified);
int ew_prepared_new(const ew_prepared* p, int departed, void** ptr, int64_t* bytes);
void ew_prepared_free(ew_prepared* p);

/* The DP group: plan_edit, NCCL communicator (owned; NULL = none) with one
 * prepared shrunk communicator per possible departure (prepare_comms: a
 * collective ncclCommSplit per member, splitShare, warmed by one
 * all-reduce), micro-batch reshaper, recovery -> MttrEvent.  kind: 0
 * FailStop, 2 ScaleIn, 3 ScaleOut (elaskit::EventKind).  prepare_comms: bit
 * 0 prepares the communicators, bit 1 builds them with splitShare (less
 * memory; NCCL then forbids concurrent use of siblings).  old_buf / replica /
 * new_buf are used when no prepared recovery is attached (planning at failure
 * time).  ScaleOut (the reference's rejoin, sim.cpp:608,676-677 with
 * comm_edit_time sim.cpp:436-450): `departed` lists the joiners; every
 * member (old_buf = its shard, new_buf) and every joiner (new_buf only)
 * calls recover; a
 * joiner's group comes from ew_dp_group_create_joiner (the members' group
 * channel name and current members, `me` outside them).
 * ew_dp_group_prepare_join: steady-state grown communicator over members +
 * joiners (collective over both), so the join's comm repair is a lookup. */
typedef struct ew_dp_group ew_dp_group;
int ew_dp_group_create(ew_channel* ch, const int64_t* layer_bytes, int n_layers, ew_comm* comm,
                       int per_slot_mbs, int num_microbatches, int64_t block_bytes,
                       int prepare_comms, ew_dp_group** out);
int ew_dp_group_create_joiner(ew_store* store, const char* group_name, const int64_t* layer_bytes,
                              int n_layers, const int* members, int n_members, int me,
                              int per_slot_mbs, int num_microbatches, int64_t block_bytes,
                              ew_dp_group** out);
int ew_dp_group_prepare_join(ew_dp_group* g, const int* joiners, int n);
/* steady-state peer mapping of this member's OLD shard and replica (NULL if
 * none) and the verification arrays (collective over the members); rows:
 * the per-step snapshot rows of those buffers (NULL: re-read at the event).
 * prepare_move (local): this rank's verified program for one expected event
 * (kind 0/2 departure set, 3 joiners) into new_buf, bound in steady state. */
int ew_dp_group_premap(ew_dp_group* g, void* old_buf, void* replica, const uint64_t* old_rows,
                       const uint64_t* replica_rows);
int ew_dp_group_prepare_move(ew_dp_group* g, int kind, const int* targets, int n, void* new_buf);
int ew_dp_group_attach(ew_dp_group* g, ew_prepared* prepared);
/* the step this member's OLD shard and replica hold (SnapshotRing step_tag,
 * param_fabric.hpp:42); an event at another step fails the verdict */
int ew_dp_group_set_snapshot_step(ew_dp_group* g, int64_t step);
int ew_dp_group_prepare(ew_dp_group* g);
/* prepared communicators for the given departure sets instead (set i =
 * members[offsets[i] .. offsets[i + 1]), n_sets + 1 offsets) */
int ew_dp_group_prepare_sets(ew_dp_group* g, const int* members, const int* offsets, int n_sets);
int ew_dp_group_recover(ew_dp_group* g, const int* departed, int n, int kind, void* old_buf,
                        void* replica, void* new_buf, int step, ew_stream_t stream,
                        ew_mttr_event* ev);
int ew_dp_group_comm(const ew_dp_group* g, ew_comm** comm); /* borrowed */
int ew_dp_group_members(const ew_dp_group* g, int* out, int cap, int* n);
int ew_dp_group_microbatches(const ew_dp_group* g, int* out, int cap, int* n);
void ew_dp_group_free(ew_dp_group* g);

/* Heartbeat failure detector of a node's DP group (recovery.hpp
 * FailureDetector; replaces the reference's constant detect_s,
 * presets.hpp:63 as charged at sim.cpp:601): collective create over the channel; each member beats
 * every period_s once its GPU completed a tiny piece of work; a member
 * silent for timeout_s is failed.  wait: up to max_wait_s for a failure;
 * *n = 0 if none; *detect_s = seconds from the failed member's last beat to
 * the verdict.  stop: this member stops beating (fault injection). */
typedef struct ew_detector ew_detector;
int ew_detector_create(ew_channel* ch, const char* tag, double period_s, double timeout_s,
                       ew_detector** out);
int ew_detector_failed(const ew_detector* d, int* out, int cap, int* n);
int ew_detector_wait(const ew_detector* d, double max_wait_s, int* out, int cap, int* n,
                     double* detect_s);
int ew_detector_stop(ew_detector* d);
void ew_detector_free(ew_detector* d);

/* Staged in-place reshard executor (config D): collective over a channel of
 * old + new members; buf holds OLD on entry and NEW on exit. */
typedef struct ew_inplace_exec ew_inplace_exec;
int ew_inplace_exec_create(ew_channel* ch, const int64_t* layer_bytes, int n_layers,
                           const int* old_members, int n_old, const int* new_members, int n_new,
                           void* buf, void* replica, int64_t stage_bytes, int64_t phase_bytes,
                           int slack, int gather_streams, int flush_ctas, int64_t block_bytes,
                           double barrier_timeout_s, ew_inplace_exec** out);
int ew_inplace_exec_launch(ew_inplace_exec* x, uint64_t* block_sums, ew_stream_t stream);
int ew_inplace_exec_timed_out(const ew_inplace_exec* x, int* timed_out);
int ew_inplace_exec_info(const ew_inplace_exec* x, int64_t* n_phases, int64_t* stage_alloc);
void ew_inplace_exec_free(ew_inplace_exec* x);

/* Ring replicas (recovery.hpp ReplayReplica / RingReplica), collective over
 * a channel of the ring's members.  Replay: the holder applies the owner's
 * AdamW step to its replica with the owner's gradient shard read from peer
 * memory (ew_adam_step_rows, replica rows in the same pass); verify compares
 * those rows with the owner's (reread != 0: recompute the replica's rows from
 * HBM).  Ring: the holder pulls the owner's snapshot and verifies it against
 * the owner's rows.  *bad_count (device u32) = mismatching rows. */
typedef struct ew_replay_replica ew_replay_replica;
int ew_replay_replica_create(ew_channel* ch, const float* my_grad, const uint64_t* my_rows,
                             float* master, float* exp_avg, float* exp_avg_sq,
                             uint16_t* param_bf16, int64_t n, const void* image,
                             int64_t image_bytes, int64_t block_bytes, ew_replay_replica** out);
int ew_replay_replica_replay(ew_replay_replica* r, const ew_adam_hyper* hyper, int64_t step,
                             ew_stream_t stream);
int ew_replay_replica_verify(const ew_replay_replica* r, uint32_t* bad_count, int reread,
                             ew_stream_t stream);
int ew_replay_replica_owner(const ew_replay_replica* r, int* owner);
void ew_replay_replica_free(ew_replay_replica* r);
typedef struct ew_ring_replica ew_ring_replica;
int ew_ring_replica_create(ew_channel* ch, const ew_layout* layout, const void* my_snap,
                           const uint64_t* my_rows, void* replica, int64_t block_bytes,
                           ew_ring_replica** out);
int ew_ring_replica_refresh(const ew_ring_replica* r, uint32_t* bad_count, ew_stream_t stream);
void ew_ring_replica_free(ew_ring_replica* r);

/* (d) fused with its collective over peer memory, through the rendezvous
 * (recovery.hpp PeerReduce): collective over a channel; each rank passes its
 * own units (or its int64 accumulator) and output; the library exchanges the
 * IPC handles and weights, builds the peer fold and a device barrier.
 * scale(): local absmax, max over ranks (one double each over the channel),
 * fixed-point bits of the global unit set (synchronises the stream once).
 * run(): barrier -> reduce-scatter -> barrier -> all-gather, stream-ordered.
 * wait(): a trailing barrier before any rank frees its buffers. */
typedef struct ew_peer_reduce ew_peer_reduce;
int ew_peer_reduce_create(ew_channel* ch, const float* const* units, const double* weights,
                          int n_units, float* out, int64_t n, double barrier_timeout_s,
                          ew_peer_reduce** handle);
int ew_peer_reduce_create_i64(ew_channel* ch, const int64_t* acc, float* out, int64_t n,
                              double barrier_timeout_s, ew_peer_reduce** handle);
int ew_peer_reduce_scale(ew_peer_reduce* r, ew_stream_t stream, int* frac_bits);
int ew_peer_reduce_run(ew_peer_reduce* r, int frac_bits, ew_stream_t stream);
int ew_peer_reduce_wait(ew_peer_reduce* r, ew_stream_t stream);
int ew_peer_reduce_info(const ew_peer_reduce* r, int64_t* total_units, int* timed_out);
void ew_peer_reduce_free(ew_peer_reduce* r);

/* Host-memory images (recovery.hpp HostImages, the H2D_D2D medium): one
 * double-buffered POSIX shm image per member, pinned for this GPU unless
 * map_for_device == 0; collective over the channel.  publish(): D2H into the
 * slot of `epoch` (-1: next) then the commit word, stream-ordered.
 * device_ptr(): the member's last committed image (for a copy-table slot). */
typedef struct ew_host_images ew_host_images;
int ew_host_images_create(ew_channel* ch, const ew_layout* layout, const char* tag,
                          const int* readable, int n_readable, int map_for_device,
                          ew_host_images** out);
int ew_host_images_publish(ew_host_images* h, const void* live, int64_t epoch, ew_stream_t stream,
                           int64_t* epoch_out);
int ew_host_images_commit_host(ew_host_images* h, int64_t epoch);
int ew_host_images_committed(const ew_host_images* h, int member, int64_t* epoch);
int ew_host_images_device_ptr(const ew_host_images* h, int member, void** ptr);
int ew_host_images_host_ptr(const ew_host_images* h, int member, int64_t epoch, void** ptr,
                            int64_t* bytes);
void ew_host_images_free(ew_host_images* h);

/* Non-blocking layer migration with shadow-gradient payback (recovery.hpp
 * LayerMigration), collective over a channel of exactly {source, target}.
 * step(): 0 pull_params (target), 1 shadow_done (source), 2 prefetch_payback
 * (target: waits for shadow_done, pulls the source's accumulator), 3 payback
 * (target, unoverlapped acc += peer acc).  run(): the target's (target_side
 * != 0) or the shadow's whole schedule for M micro-batch units. */
typedef struct ew_layer_migration ew_layer_migration;
int ew_layer_migration_create(ew_channel* ch, int source, int target, void* params,
                              int64_t param_bytes, int64_t* acc, int64_t n, int transfer_ctas,
                              double barrier_timeout_s, ew_layer_migration** out);
int ew_layer_migration_step(ew_layer_migration* m, int what, ew_stream_t stream);
int ew_layer_migration_run(ew_layer_migration* m, int target_side, const float* const* units,
                           const double* weights, int n_units, int64_t n, int frac_bits, int k,
                           ew_stream_t compute, ew_stream_t transfer);
int ew_layer_migration_info(const ew_layer_migration* m, const int64_t** payback_buffer,
                            int* timed_out);
void ew_layer_migration_free(ew_layer_migration* m);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* EW_API_H */
