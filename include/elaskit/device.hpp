// C++ convenience layer over the device half of include/ew_api.h.
//
// Header-only RAII wrappers that throw the reference's exception types
// (CoverageMismatch, MissingBackup, ...) instead of returning ew_status, so a
// C++ executor written against the elaskit headers can drive the sm_100a
// kernels in the same style as the planners.  Device pointers are raw; the
// caller owns the memory and the stream.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "elaskit/b200.hpp"
#include "elaskit/communicator.hpp"
#include "elaskit/dataflow.hpp"
#include "elaskit/migration.hpp"
#include "elaskit/param_fabric.hpp"
#include "elaskit/rng.hpp"
#include "ew_api.h"

namespace elaskit::device {

struct CudaError final : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Rethrow an ew_status as the reference exception it stands for.
inline void check(int status) {
  if (status == EW_OK) return;
  const std::string msg = ew_last_error();
  switch (status) {
    case EW_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case EW_ERR_COVERAGE_MISMATCH: throw CoverageMismatch(msg);
    case EW_ERR_MISSING_BACKUP: throw MissingBackup(msg);
    case EW_ERR_NO_SURVIVORS: throw NoSurvivors(msg);
    case EW_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case EW_ERR_MISMATCHED_DP: throw MismatchedDpDegree(msg);
    case EW_ERR_DISCONNECTED: throw DisconnectedGroup(msg);
    case EW_ERR_INSUFFICIENT_MEMORY: throw InsufficientTargetMemory(msg);
    case EW_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case EW_ERR_CUDA:
    case EW_ERR_NCCL: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

// Segment map of one rank's packed shard, resident on the current device.
class ShardMap {
 public:
  ShardMap(const PartitionLayout& layout, int rank, std::int64_t block_bytes = 65536) {
    std::vector<ew_segment> segs;
    for (const b200::Segment& s : b200::shard_segments(layout, rank))
      segs.push_back({s.global_lo, s.length, s.local_off});
    check(ew_shardmap_create(segs.data(), static_cast<std::int64_t>(segs.size()), block_bytes,
                             &map_));
  }
  ~ShardMap() { ew_shardmap_free(map_); }
  ShardMap(const ShardMap&) = delete;
  ShardMap& operator=(const ShardMap&) = delete;

  std::int64_t bytes() const { return ew_shardmap_bytes(map_); }
  std::int64_t rows() const { return ew_shardmap_num_rows(map_); }
  const ew_shardmap* get() const { return map_; }

  // snap <- live, row_sums <- checksum rows of live (device uint64[2*rows()]).
  void snapshot(const void* live, void* snap, std::uint64_t* row_sums, ew_stream_t s) const {
    check(ew_snapshot(map_, live, snap, row_sums, s));
  }
  void verify(const void* buf, const std::uint64_t* expected, std::uint32_t* bad_count,
              ew_stream_t s) const {
    check(ew_verify(map_, buf, expected, bad_count, nullptr, 0, s));
  }

 private:
  ew_shardmap* map_ = nullptr;
};

// One GPU's reshard program: TransferPlan -> copies -> resolved pointers.
class CopyProgram {
 public:
  // table[role * table_ranks + rank]: local or IPC-mapped buffer pointers.
  // verify_map (NEW's segment map on exec_rank, pull programs): the copy
  // also checksums what it lands — see launch(s, block_sums).
  CopyProgram(const std::vector<b200::CopyDesc>& copies, const std::vector<void*>& table,
              int table_ranks, int exec_rank, const ShardMap* verify_map = nullptr) {
    std::vector<ew_copy_desc> d;
    d.reserve(copies.size());
    for (const b200::CopyDesc& c : copies)
      d.push_back({static_cast<std::int32_t>(c.src_role), c.src_rank,
                   static_cast<std::int32_t>(c.dst_role), c.dst_rank, c.src_off, c.dst_off,
                   c.bytes});
    if (verify_map != nullptr)
      check(ew_copy_program_create_verified(d.data(), static_cast<std::int64_t>(d.size()),
                                            table.data(), table_ranks, exec_rank,
                                            verify_map->get(), &prog_));
    else
      check(ew_copy_program_create(d.data(), static_cast<std::int64_t>(d.size()), table.data(),
                                   table_ranks, exec_rank, &prog_));
  }
  ~CopyProgram() { ew_copy_program_free(prog_); }
  CopyProgram(const CopyProgram&) = delete;
  CopyProgram& operator=(const CopyProgram&) = delete;

  void launch(ew_stream_t s, int n_ctas = 0, int remote_ctas = 0) const {
    check(ew_copy_program_launch(prog_, n_ctas, remote_ctas, s));
  }
  // Verified programs: add the landed bytes' block checksums to block_sums
  // (device u64 [2 * num_blocks()], zeroed by the caller).
  void launch(ew_stream_t s, std::uint64_t* block_sums, int n_ctas = 0,
              int remote_ctas = 0) const {
    check(ew_copy_program_launch_verified(prog_, n_ctas, remote_ctas, block_sums, s));
  }
  std::int64_t num_blocks() const {
    std::int64_t n = 0;
    check(ew_copy_program_num_blocks(prog_, &n));
    return n;
  }

 private:
  ew_copy_program* prog_ = nullptr;
};

// A host range pinned and mapped for the copy kernels (Medium::H2D_D2D
// sources: a departed rank's image in node-shared host memory).  device()
// goes into a CopyProgram table slot like any peer pointer.
class HostRegistration {
 public:
  HostRegistration(void* host, std::int64_t bytes) : host_(host) {
    check(ew_host_register(host, bytes, &dev_));
  }
  ~HostRegistration() {
    if (host_ != nullptr) ew_host_unregister(host_);
  }
  HostRegistration(const HostRegistration&) = delete;
  HostRegistration& operator=(const HostRegistration&) = delete;
  void* device() const { return dev_; }

 private:
  void* host_ = nullptr;
  void* dev_ = nullptr;
};

// Dropout keep-bits for samples [sample_lo, sample_lo + n_samples) of one
// (layer, op) stream — the masks the reference derives from draw().
inline void dropout_mask(std::uint64_t seed, std::uint64_t sample_lo, std::int64_t n_samples,
                         std::uint32_t layer, std::uint32_t op, std::int64_t n_elems, double keep,
                         std::uint32_t* bits, ew_stream_t s) {
  check(ew_philox_dropout_mask(seed, sample_lo, n_samples, layer, op, n_elems, keep, bits, s));
}

}  // namespace elaskit::device
