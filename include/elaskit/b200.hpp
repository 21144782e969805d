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
#include <map>
#include <set>
#include <utility>
#include <vector>

#include "elaskit/cluster.hpp"
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

// Replica-aware sourcing of a PULL program (a B200 executor option, off by
// default): every exec_rank keeps a current ring replica of the member it
// backs up (SnapshotRing::backs_up, kept byte-identical each step by the
// replay replica and verified by its rows), so copies the plan sources from
// that member's OLD shard can read exec_rank's own replica instead — same
// bytes, same source offsets (the replica is packed like the owner's shard),
// local HBM instead of NVLink.  The plan, the landed layout and the
// verification are unchanged; only the physical source moves.  Config B 8->7
// drop r3: the bottleneck GPU's NVLink bytes fall from 10.11 to 6.74 GB;
// drop r7 and 4->3 drop r3 become all-local.
std::vector<CopyDesc> prefer_local_replica(const std::vector<CopyDesc>& pull_copies,
                                           const SnapshotRing& ring, const std::set<int>& failed,
                                           int exec_rank);

// Staged in-place reshard (state that fills HBM).
// Each rank keeps ONE buffer that holds its OLD shard on entry and its NEW
// shard on exit; the move runs in phases over the global byte space.  Phases
// are cut only where every rank that keeps its OLD bytes in place has
// new_prefix(G) >= old_prefix(G) (departures, phases run downwards) or <=
// (joins, upwards), so the OLD bytes later phases read lie beyond each
// phase's NEW range.  Per phase and rank, `direct` is the part of the NEW
// range clear of the OLD bytes phases j-slack .. j still read (written in
// place by gather_j once every rank finished gather_{j-slack-1}) and
// `staged` the rest (gathered into a staging buffer, flushed after the
// phase's cross-GPU barrier).  Offsets are packed NEW offsets; phases are
// global [lo, hi) in processing order.
using ByteRange = std::pair<std::int64_t, std::int64_t>;

struct InPlaceRanges {
  std::vector<ByteRange> cut, direct, staged;  // one per phase
};

struct InPlaceSchedule {
  bool descending = true;
  int slack = 1;
  int ring = 3;                          // staging buffers in rotation (slack + 2)
  std::vector<ByteRange> phases;         // global ranges, processing order
  std::map<int, InPlaceRanges> ranks;    // every member of the target layout
  std::vector<int> holders;              // members whose OLD is read in place
  std::int64_t stage_alloc = 0;          // bytes per staging buffer (0: none)
};

// Greedy phases over the safe cut points (layer boundaries of layer_bytes,
// plus points inside a layer that pass the prefix test), each as large as
// phase_bytes of NEW per rank and stage_bytes of staged bytes allow.
// Throws std::invalid_argument when shards neither all grow nor all shrink,
// CoverageMismatch if check_inplace fails (it is run before returning).
InPlaceSchedule inplace_schedule(const std::vector<std::int64_t>& layer_bytes,
                                 const PartitionLayout& src, const PartitionLayout& dst,
                                 const std::set<int>& failed, std::int64_t stage_bytes,
                                 std::int64_t phase_bytes, int slack);

// Rank's pull copies restricted to NEW offsets [lo, hi), destination offsets
// moved by -lo + shift (the staged part of a phase: shift = lo % 16 into a
// staging buffer; the direct part: shift = lo keeps NEW's own offsets).
std::vector<CopyDesc> clip_copies(const std::vector<CopyDesc>& copies, std::int64_t lo,
                                  std::int64_t hi, std::int64_t shift);

// Every write against every read it could race with: gather_j's direct
// writes vs the OLD reads of phases >= j - slack, flush_j's writes vs the
// reads of phases > j.  Throws CoverageMismatch naming the first overlap.
void check_inplace(const InPlaceSchedule& s, const PartitionLayout& src);

// One stage's DP membership change under one event — the input of the
// recovery path: old = dp_group(state, stage), next = apply_event(state, ev),
// members = dp_group(next, stage) (empty when the stage emptied: EmptyStage
// is the graph planner's case, not a DP reshard), departed = old \ members
// (the `failed` set of integrity_check / overlap_matrix), slow = members whose
// slow_factor changed.  ScaleOut arrivals wait in next.free_pool until a
// placement puts them in the grid, so a pure ScaleOut yields no change here.
struct DpTransition {
  ClusterState next;
  std::vector<DeviceId> old_members, members;
  std::set<int> departed;
  std::vector<DeviceId> slow;
};

DpTransition dp_transition(const ClusterState& state, const ElasticEvent& ev, int stage);

// Sample offsets of micro-batch 0 whose owning slot changes between two
// assignments — the SampleReassignment list recover_elaswave derives before
// reshard_rng (reference: sim.cpp:694-715; offsets beyond the smaller
// per-micro-batch total are ignored, as there).
std::vector<SampleReassignment> sample_reassignments(const MicrobatchAssignment& old_mb,
                                                     const MicrobatchAssignment& new_mb);

}  // namespace elaskit::b200
