// B200-build additions to the elaskit planning API.
//
// The reference never composes an interleaved PartitionLayout and never
// executes a TransferPlan.  These helpers do both
// on the host: they turn ZeroLayout ownership into the PartitionLayout that
// overlap_matrix consumes, give each rank's packed shard buffer its
// local<->global segment map, and lower a TransferPlan into per-GPU copy
// descriptors that the sm_100a reshard kernel executes.
#pragma once

#include <cstdint>
#include <set>
#include <vector>

#include "elaskit/dataflow.hpp"
#include "elaskit/migration.hpp"
#include "elaskit/param_fabric.hpp"
#include "elaskit/rng.hpp"

namespace elaskit::b200 {

// Interleaved ZeRO as a PartitionLayout: for every layer l in order and every
// rank index j of the ascending `ranks`, rank ranks[j] owns
// layer_offset(l) + shard(l, j) when non-empty (ownership rule of reference
// migration.cpp:73-77; composition per SURVEY §8(a) A4).  Requires
// z.kind == Interleaved; the DP degree is ranks.size() (z.dp_degree is
// ignored so one ZeroLayout can be laid over any survivor set).
PartitionLayout interleaved_layout(const ZeroLayout& z, const std::vector<int>& ranks);

// One interval of a rank's packed shard buffer: bytes
// [global_lo, global_lo + length) of the flat space live at
// [local_off, local_off + length) of the rank's buffer.  Intervals are packed
// back to back in ascending global order.
struct Segment {
  std::int64_t global_lo = 0;
  std::int64_t length = 0;
  std::int64_t local_off = 0;
};

std::vector<Segment> shard_segments(const PartitionLayout& layout, int rank);
std::int64_t shard_bytes(const PartitionLayout& layout, int rank);

// Buffers a reshard touches on rank r:
//   Old     - r's packed shard under the source layout (its live state),
//   Replica - r's ring copy of the rank it backs up (SnapshotRing::backs_up),
//             packed in that rank's source layout,
//   New     - r's packed shard under the target layout.
enum class BufRole : int { Old = 0, Replica = 1, New = 2 };

struct CopyDesc {
  BufRole src_role = BufRole::Old;
  int src_rank = -1;  // GPU that holds the source buffer
  BufRole dst_role = BufRole::New;
  int dst_rank = -1;  // GPU that holds the destination buffer
  std::int64_t src_off = 0;
  std::int64_t dst_off = 0;
  std::int64_t bytes = 0;
};

// Lowers `plan` (= overlap_matrix(src, dst, failed, ring)) into the copies one
// GPU issues.  push: copies whose source buffer is on exec_rank (remote
// stores); pull: copies whose destination is exec_rank (remote loads).  Both
// include exec_rank's retained bytes (owner unchanged, which overlap_matrix
// leaves out but the packed position may still change).  Throws
// CoverageMismatch if the plan does not belong to the layouts.
std::vector<CopyDesc> reshard_copies(const TransferPlan& plan, const PartitionLayout& src,
                                     const PartitionLayout& dst, const std::set<int>& failed,
                                     const SnapshotRing* ring, int exec_rank, bool push);

// Sample offsets of micro-batch 0 whose owning slot changes between two
// assignments — the SampleReassignment list recover_elaswave derives before
// reshard_rng (reference: sim.cpp:694-715; offsets beyond the smaller
// per-micro-batch total are ignored, as there).
std::vector<SampleReassignment> sample_reassignments(const MicrobatchAssignment& old_mb,
                                                     const MicrobatchAssignment& new_mb);

}  // namespace elaskit::b200
