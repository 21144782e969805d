// Interleaved-ZeRO layout composer and TransferPlan lowering (host side).
#include <algorithm>
#include <map>
#include <string>

#include "elaskit/b200.hpp"

namespace elaskit::b200 {

PartitionLayout interleaved_layout(const ZeroLayout& z, const std::vector<int>& ranks) {
  if (z.kind != ZeroKind::Interleaved)
    throw std::invalid_argument("interleaved_layout needs ZeroKind::Interleaved");
  if (ranks.empty()) throw std::invalid_argument("interleaved_layout needs at least one rank");
  std::vector<int> order(ranks);
  std::sort(order.begin(), order.end());
  if (std::adjacent_find(order.begin(), order.end()) != order.end())
    throw std::invalid_argument("interleaved_layout: duplicate rank");

  ZeroLayout over = z;
  over.dp_degree = static_cast<int>(order.size());
  PartitionLayout out;
  out.total_bytes = over.total_bytes();
  for (const int r : order) out.ranges[r];
  std::int64_t base = 0;
  for (std::size_t l = 0; l < over.layer_bytes.size(); ++l) {
    if (over.layer_bytes[l] < 0) throw std::invalid_argument("negative layer size");
    for (std::size_t j = 0; j < order.size(); ++j) {
      const ByteInterval s = over.shard(static_cast<int>(l), static_cast<int>(j));
      if (s.size() > 0) out.ranges[order[j]].push_back({base + s.lo, base + s.hi});
    }
    base += over.layer_bytes[l];
  }
  return out;
}

std::vector<Segment> shard_segments(const PartitionLayout& layout, int rank) {
  std::vector<Segment> segs;
  const auto it = layout.ranges.find(rank);
  if (it == layout.ranges.end()) return segs;
  std::int64_t local = 0;
  segs.reserve(it->second.size());
  for (const ByteInterval& iv : it->second) {
    segs.push_back({iv.lo, iv.size(), local});
    local += iv.size();
  }
  return segs;
}

std::int64_t shard_bytes(const PartitionLayout& layout, int rank) {
  std::int64_t n = 0;
  const auto it = layout.ranges.find(rank);
  if (it != layout.ranges.end())
    for (const ByteInterval& iv : it->second) n += iv.size();
  return n;
}

namespace {

// Local offset of global byte range [lo, hi) inside `rank`'s packed buffer;
// the range must sit inside one of the rank's intervals.
class LocalIndex {
 public:
  explicit LocalIndex(const PartitionLayout& layout) {
    for (const auto& [rank, ivs] : layout.ranges) {
      auto& v = index_[rank];
      std::int64_t local = 0;
      for (const ByteInterval& iv : ivs) {
        v.push_back({iv.lo, iv.hi, local});
        local += iv.size();
      }
    }
  }

  std::int64_t offset(int rank, std::int64_t lo, std::int64_t hi) const {
    const auto it = index_.find(rank);
    if (it != index_.end()) {
      const auto& v = it->second;
      auto pos = std::upper_bound(v.begin(), v.end(), lo,
                                  [](std::int64_t x, const Row& r) { return x < r.lo; });
      if (pos != v.begin()) {
        const Row& r = *(pos - 1);
        if (lo >= r.lo && hi <= r.hi) return r.local + (lo - r.lo);
      }
    }
    throw CoverageMismatch("bytes [" + std::to_string(lo) + "," + std::to_string(hi) +
                           ") are not held by rank " + std::to_string(rank));
  }

 private:
  struct Row {
    std::int64_t lo, hi, local;
  };
  std::map<int, std::vector<Row>> index_;
};

// Owner of [lo,hi) under `layout` (the range lies inside one interval).
int owner_of_range(const PartitionLayout& layout, std::int64_t lo) {
  for (const auto& [rank, ivs] : layout.ranges) {
    auto pos = std::upper_bound(ivs.begin(), ivs.end(), lo,
                                [](std::int64_t x, const ByteInterval& iv) { return x < iv.lo; });
    if (pos != ivs.begin() && lo < (pos - 1)->hi) return rank;
  }
  return -1;
}

}  // namespace

std::vector<CopyDesc> reshard_copies(const TransferPlan& plan, const PartitionLayout& src,
                                     const PartitionLayout& dst, const std::set<int>& failed,
                                     const SnapshotRing* ring, int exec_rank, bool push) {
  const LocalIndex old_index(src);
  const LocalIndex new_index(dst);
  std::vector<CopyDesc> out;

  for (const TransferEntry& e : plan.entries) {
    const bool from_replica = e.medium == Medium::H2D_D2D;
    const bool mine = push ? (e.src_rank == exec_rank) : (e.dst_rank == exec_rank);
    if (!mine) continue;
    CopyDesc c;
    c.src_rank = e.src_rank;
    c.dst_rank = e.dst_rank;
    c.dst_role = BufRole::New;
    c.bytes = e.iv.size();
    c.dst_off = new_index.offset(e.dst_rank, e.iv.lo, e.iv.hi);
    if (from_replica) {
      // the holder's replica is packed like the dead owner's old shard
      const int owner = owner_of_range(src, e.iv.lo);
      if (owner < 0 || !failed.contains(owner) || ring == nullptr ||
          ring->backed_up_by(owner) != e.src_rank)
        throw CoverageMismatch("h2d_d2d entry at byte " + std::to_string(e.iv.lo) +
                               " does not come from a failed owner's ring holder");
      c.src_role = BufRole::Replica;
      c.src_off = old_index.offset(owner, e.iv.lo, e.iv.hi);
    } else {
      c.src_role = BufRole::Old;
      c.src_off = old_index.offset(e.src_rank, e.iv.lo, e.iv.hi);
    }
    out.push_back(c);
  }

  // retained bytes: exec_rank keeps ownership but its packing may change
  const auto a = src.ranges.find(exec_rank);
  const auto b = dst.ranges.find(exec_rank);
  if (a != src.ranges.end() && b != dst.ranges.end() && !failed.contains(exec_rank)) {
    std::size_t i = 0, j = 0;
    const auto& x = a->second;
    const auto& y = b->second;
    while (i < x.size() && j < y.size()) {
      const std::int64_t lo = std::max(x[i].lo, y[j].lo);
      const std::int64_t hi = std::min(x[i].hi, y[j].hi);
      if (lo < hi) {
        CopyDesc c;
        c.src_role = BufRole::Old;
        c.src_rank = exec_rank;
        c.dst_role = BufRole::New;
        c.dst_rank = exec_rank;
        c.src_off = old_index.offset(exec_rank, lo, hi);
        c.dst_off = new_index.offset(exec_rank, lo, hi);
        c.bytes = hi - lo;
        out.push_back(c);
      }
      if (x[i].hi <= y[j].hi) ++i;
      else ++j;
    }
  }
  return out;
}

std::vector<SampleReassignment> sample_reassignments(const MicrobatchAssignment& old_mb,
                                                     const MicrobatchAssignment& new_mb) {
  const auto slot_at = [](const MicrobatchAssignment& a,
                          const std::vector<std::pair<std::int64_t, std::int64_t>>& ranges,
                          std::int64_t off) {
    for (std::size_t i = 0; i < ranges.size(); ++i)
      if (off >= ranges[i].first && off < ranges[i].second) return a.slots[i];
    return -1;
  };
  const auto old_ranges = old_mb.sample_ranges(0, 0);
  const auto new_ranges = new_mb.sample_ranges(0, 0);
  const int total = std::min(old_mb.samples_per_microbatch(), new_mb.samples_per_microbatch());
  std::vector<SampleReassignment> out;
  for (int off = 0; off < total; ++off) {
    const int from = slot_at(old_mb, old_ranges, off);
    const int to = slot_at(new_mb, new_ranges, off);
    if (from != to && from >= 0 && to >= 0)
      out.push_back({static_cast<std::int64_t>(off), from, to});
  }
  return out;
}

// The recovery path's input from the cluster model (SURVEY §8(a) A17:
// ElasticEvent feeds plan_edit; the survivor set feeds the layouts).
DpTransition dp_transition(const ClusterState& state, const ElasticEvent& ev, int stage) {
  DpTransition t;
  t.old_members = dp_group(state, stage);
  t.next = apply_event(state, ev);
  try {
    t.members = dp_group(t.next, stage);
  } catch (const EmptyStage&) {
    t.members.clear();
  }
  for (const DeviceId d : t.old_members) {
    if (std::find(t.members.begin(), t.members.end(), d) == t.members.end())
      t.departed.insert(d);
    else if (t.next.devices.at(d).slow_factor != state.devices.at(d).slow_factor)
      t.slow.push_back(d);
  }
  return t;
}

std::vector<CopyDesc> prefer_local_replica(const std::vector<CopyDesc>& pull_copies,
                                           const SnapshotRing& ring, const std::set<int>& failed,
                                           int exec_rank) {
  std::vector<CopyDesc> out = pull_copies;
  if (ring.members.size() < 2 ||
      std::find(ring.members.begin(), ring.members.end(), exec_rank) == ring.members.end())
    return out;
  const int held = ring.backs_up(exec_rank);
  if (held == exec_rank || failed.count(held)) return out;  // a departed owner is sourced so already
  for (CopyDesc& c : out)
    if (c.dst_rank == exec_rank && c.src_role == BufRole::Old && c.src_rank == held) {
      c.src_role = BufRole::Replica;  // same packing, same offsets
      c.src_rank = exec_rank;
    }
  return out;
}

}  // namespace elaskit::b200
