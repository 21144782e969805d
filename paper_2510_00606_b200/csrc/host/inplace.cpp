// Staged in-place reshard schedule (elaskit/b200.hpp inplace_schedule).
//
// The reference never executes a remap (remap_time, sim.cpp:452-483, models
// it); its plan is overlap_matrix (param_fabric.cpp:82-121).  On a B200 that
// is full of state OLD, the ring replica and NEW do
// not fit side by side, so OLD and NEW share one buffer and the plan's copies
// are cut into phases whose writes never land on OLD bytes still to be read.
#include <algorithm>
#include <stdexcept>
#include <string>

#include "elaskit/b200.hpp"

namespace elaskit::b200 {
namespace {

// Packed bytes of one rank's intervals that lie below a global position.
class Prefix {
 public:
  Prefix() = default;
  explicit Prefix(const std::vector<Segment>& segs) {
    for (const Segment& s : segs) {
      lo_.push_back(s.global_lo);
      len_.push_back(s.length);
      off_.push_back(s.local_off);
    }
  }
  std::int64_t operator()(std::int64_t g) const {
    const auto it = std::lower_bound(lo_.begin(), lo_.end(), g);  // first lo >= g
    if (it == lo_.begin()) return 0;
    const std::size_t i = static_cast<std::size_t>(it - lo_.begin()) - 1;
    return off_[i] + std::min(len_[i], g - lo_[i]);
  }

 private:
  std::vector<std::int64_t> lo_, len_, off_;
};

bool overlaps(const ByteRange& a, const ByteRange& b) {
  return a.first < a.second && b.first < b.second && a.first < b.second && b.first < a.second;
}

}  // namespace

InPlaceSchedule inplace_schedule(const std::vector<std::int64_t>& layer_bytes,
                                 const PartitionLayout& src, const PartitionLayout& dst,
                                 const std::set<int>& failed, std::int64_t stage_bytes,
                                 std::int64_t phase_bytes, int slack) {
  if (stage_bytes <= 0 || phase_bytes <= 0 || slack < 0)
    throw std::invalid_argument("inplace_schedule: stage/phase bytes > 0 and slack >= 0");
  std::int64_t total = 0;
  for (const std::int64_t b : layer_bytes) total += b;
  if (total != src.total_bytes || total != dst.total_bytes)
    throw CoverageMismatch("inplace_schedule: layer bytes do not match the layouts");

  InPlaceSchedule s;
  s.slack = slack;
  s.ring = slack + 2;
  std::vector<int> execs;
  for (const auto& [r, ivs] : dst.ranges) execs.push_back(r);
  std::map<int, Prefix> newp, oldp;
  std::map<int, std::int64_t> n_old;
  for (const int r : execs) {
    newp[r] = Prefix(shard_segments(dst, r));
    if (src.ranges.count(r) && !failed.count(r)) {
      s.holders.push_back(r);
      oldp[r] = Prefix(shard_segments(src, r));
      n_old[r] = shard_bytes(src, r);
    }
  }
  bool grow = true, shrink = true;
  for (const int r : s.holders) {
    const std::int64_t nn = shard_bytes(dst, r), no = n_old[r];
    grow = grow && nn >= no;
    shrink = shrink && nn <= no;
  }
  if (!grow && !shrink)
    throw std::invalid_argument(
        "in-place staging needs every retained shard to grow (departures) or every one to "
        "shrink (joins)");
  s.descending = grow;

  // candidate cut points: layer boundaries plus points a quarter phase of one
  // rank's share apart inside each layer; keep the ones every holder allows
  const std::int64_t n_new = std::max<std::int64_t>(1, static_cast<std::int64_t>(execs.size()));
  const std::int64_t step = std::max<std::int64_t>(4096, std::min(phase_bytes, stage_bytes) * n_new / 4);
  std::vector<std::int64_t> cand;
  std::int64_t off = 0;
  for (const std::int64_t sz : layer_bytes) {
    for (std::int64_t x = off; x < off + sz; x += step) cand.push_back(x);
    off += sz;
  }
  std::sort(cand.begin(), cand.end());
  cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
  std::vector<std::int64_t> safe{0};
  for (const std::int64_t c : cand) {
    if (c <= 0 || c >= total) continue;
    bool ok = true;
    for (const int r : s.holders) {
      const std::int64_t d = newp[r](c) - oldp[r](c);
      ok = ok && (s.descending ? d >= 0 : d <= 0);
    }
    if (ok) safe.push_back(c);
  }
  safe.push_back(total);
  std::vector<std::int64_t> order(safe);
  if (s.descending) std::reverse(order.begin(), order.end());
  std::map<int, std::vector<std::int64_t>> np_, op_;
  for (const int r : execs) {
    auto& v = np_[r];
    for (const std::int64_t g : order) v.push_back(newp[r](g));
  }
  for (const int r : s.holders) {
    auto& v = op_[r];
    for (const std::int64_t g : order) v.push_back(oldp[r](g));
  }

  // greedy phases: grow while every rank's share fits phase_bytes and its
  // staged part (below the OLD bytes phases j-slack .. j read) fits stage_bytes
  std::vector<std::size_t> bounds{0};
  auto fits = [&](std::size_t a, std::size_t b) {
    const long j = static_cast<long>(bounds.size()) - 1;
    const long k = j - slack;
    for (const int r : execs) {
      const std::int64_t lo = std::min(np_[r][a], np_[r][b]);
      const std::int64_t hi = std::max(np_[r][a], np_[r][b]);
      if (hi - lo > phase_bytes) return false;
      if (!op_.count(r)) continue;
      std::int64_t staged;
      if (s.descending) {
        const std::int64_t t = k < 0 ? n_old[r] : op_[r][bounds[static_cast<std::size_t>(k)]];
        staged = std::max<std::int64_t>(0, std::min(hi, t) - lo);
      } else {
        const std::int64_t t = k < 0 ? 0 : op_[r][bounds[static_cast<std::size_t>(k)]];
        staged = std::max<std::int64_t>(0, hi - std::max(lo, t));
      }
      if (staged > stage_bytes) return false;
    }
    return true;
  };
  while (bounds.back() + 1 < order.size()) {
    const std::size_t a = bounds.back();
    std::size_t b = a + 1;
    while (b + 1 < order.size() && fits(a, b + 1)) ++b;
    bounds.push_back(b);
    s.phases.push_back({std::min(order[a], order[b]), std::max(order[a], order[b])});
  }

  // per-rank NEW cuts and the direct / staged split
  std::int64_t biggest = 0;
  const long n = static_cast<long>(s.phases.size());
  for (const int r : execs) {
    InPlaceRanges& rr = s.ranks[r];
    for (long j = 0; j < n; ++j) {
      const ByteRange& ph = s.phases[static_cast<std::size_t>(j)];
      const std::int64_t k_lo = newp[r](ph.first), k_hi = newp[r](ph.second);
      rr.cut.push_back({k_lo, k_hi});
      if (!oldp.count(r)) {  // nobody reads this rank's buffer
        rr.staged.push_back({k_lo, k_lo});
        rr.direct.push_back({k_lo, k_hi});
        continue;
      }
      const long k = j - slack;
      if (s.descending) {
        const std::int64_t t =
            k < 0 ? n_old[r] : oldp[r](s.phases[static_cast<std::size_t>(k)].second);
        const std::int64_t m = std::min(std::max(t, k_lo), k_hi);
        rr.staged.push_back({k_lo, m});
        rr.direct.push_back({m, k_hi});
      } else {
        const std::int64_t t = k < 0 ? 0 : oldp[r](s.phases[static_cast<std::size_t>(k)].first);
        const std::int64_t m = std::max(std::min(t, k_hi), k_lo);
        rr.staged.push_back({m, k_hi});
        rr.direct.push_back({k_lo, m});
      }
      biggest = std::max(biggest, rr.staged.back().second - rr.staged.back().first);
    }
  }
  s.stage_alloc = biggest > 0 ? (biggest + 15 + 255) / 256 * 256 : 0;
  check_inplace(s, src);
  return s;
}

std::vector<CopyDesc> clip_copies(const std::vector<CopyDesc>& copies, std::int64_t lo,
                                  std::int64_t hi, std::int64_t shift) {
  std::vector<CopyDesc> out;
  for (const CopyDesc& c : copies) {
    const std::int64_t a = std::max(c.dst_off, lo), b = std::min(c.dst_off + c.bytes, hi);
    if (b <= a) continue;
    CopyDesc d = c;
    d.src_off = c.src_off + (a - c.dst_off);
    d.dst_off = a - lo + shift;
    d.bytes = b - a;
    out.push_back(d);
  }
  return out;
}

void check_inplace(const InPlaceSchedule& s, const PartitionLayout& src) {
  const long n = static_cast<long>(s.phases.size());
  for (const int r : s.holders) {
    const Prefix oldp(shard_segments(src, r));
    std::vector<ByteRange> reads;
    for (const ByteRange& ph : s.phases) reads.push_back({oldp(ph.first), oldp(ph.second)});
    const InPlaceRanges& rr = s.ranks.at(r);
    for (long j = 0; j < n; ++j) {
      const std::size_t ju = static_cast<std::size_t>(j);
      for (int what = 0; what < 2; ++what) {
        const ByteRange w = what == 0 ? rr.direct[ju] : rr.staged[ju];
        for (long k = std::max(0L, what == 0 ? j - s.slack : j + 1); k < n; ++k) {
          if (overlaps(w, reads[static_cast<std::size_t>(k)]))
            throw CoverageMismatch("in-place schedule: rank " + std::to_string(r) + " phase " +
                                   std::to_string(j) + (what == 0 ? " direct" : " staged") +
                                   " write overlaps OLD bytes phase " + std::to_string(k) +
                                   " reads");
        }
      }
    }
  }
}

}  // namespace elaskit::b200
