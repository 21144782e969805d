// C ABI over the host planners (include/ew_api.h, planning half).
//
// Every entry point runs the C++ API of include/elaskit and converts the
// reference's exception types to ew_status codes; nothing throws across the
// boundary.
#include <cstring>
#include <string>

#include "elaskit/b200.hpp"
#include "elaskit/communicator.hpp"
#include "elaskit/dataflow.hpp"
#include "elaskit/migration.hpp"
#include "elaskit/param_fabric.hpp"
#include "elaskit/rng.hpp"
#include "ew_api.h"

#include "host/guarded.hpp"

struct ew_layout {
  elaskit::PartitionLayout layout;
};

struct ew_plan {
  elaskit::TransferPlan plan;
};

struct ew_inplace {
  elaskit::b200::InPlaceSchedule s;
};

namespace {

using ew::set_error;
using ew::guarded;

std::set<int> to_set(const int* v, int n) {
  std::set<int> s;
  for (int i = 0; i < n; ++i) s.insert(v[i]);
  return s;
}

elaskit::SnapshotRing to_ring(const int* members, int n) {
  elaskit::SnapshotRing r;
  r.members.assign(members, members + n);
  return r;
}

}  // namespace

extern "C" {

int ew_layout_interleaved(const int64_t* layer_bytes, int n_layers, const int* ranks,
                          int n_ranks, ew_layout** out) {
  return guarded([&]() -> int {
    if (out == nullptr || n_layers < 0 || n_ranks < 1 || (n_layers > 0 && !layer_bytes) || !ranks)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_layout_interleaved: bad arguments");
    elaskit::ZeroLayout z;
    z.kind = elaskit::ZeroKind::Interleaved;
    z.dp_degree = n_ranks;
    z.layer_bytes.assign(layer_bytes, layer_bytes + n_layers);
    auto* l = new ew_layout{elaskit::b200::interleaved_layout(z, std::vector<int>(ranks, ranks + n_ranks))};
    *out = l;
    return EW_OK;
  });
}

int ew_layout_contiguous(const int* ranks, int n_ranks, int64_t total, ew_layout** out) {
  return guarded([&]() -> int {
    if (out == nullptr || n_ranks < 0 || (n_ranks > 0 && !ranks))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_layout_contiguous: bad arguments");
    *out = new ew_layout{elaskit::contiguous_layout(std::vector<int>(ranks, ranks + n_ranks), total)};
    return EW_OK;
  });
}

int ew_layout_from_intervals(const int* ranks, const int* counts, int n_ranks,
                             const ew_interval* ivs, int64_t total, ew_layout** out) {
  return guarded([&]() -> int {
    if (out == nullptr || n_ranks < 0 || (n_ranks > 0 && (!ranks || !counts)))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_layout_from_intervals: bad arguments");
    auto* l = new ew_layout();
    l->layout.total_bytes = total;
    int64_t k = 0;
    for (int i = 0; i < n_ranks; ++i) {
      auto& list = l->layout.ranges[ranks[i]];
      for (int c = 0; c < counts[i]; ++c, ++k) list.push_back({ivs[k].lo, ivs[k].hi});
    }
    *out = l;
    return EW_OK;
  });
}

void ew_layout_free(ew_layout* layout) { delete layout; }

int64_t ew_layout_total_bytes(const ew_layout* layout) {
  return layout ? layout->layout.total_bytes : -1;
}

int ew_layout_num_ranks(const ew_layout* layout) {
  return layout ? static_cast<int>(layout->layout.ranges.size()) : -1;
}

int ew_layout_ranks(const ew_layout* layout, int* out, int cap) {
  if (layout == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL layout");
  if (cap < static_cast<int>(layout->layout.ranges.size()))
    return set_error(EW_ERR_CAPACITY, "rank buffer too small");
  int i = 0;
  for (const auto& kv : layout->layout.ranges) out[i++] = kv.first;
  return EW_OK;
}

int64_t ew_layout_shard_bytes(const ew_layout* layout, int rank) {
  return layout ? elaskit::b200::shard_bytes(layout->layout, rank) : -1;
}

int64_t ew_layout_num_segments(const ew_layout* layout, int rank) {
  if (layout == nullptr) return -1;
  const auto it = layout->layout.ranges.find(rank);
  return it == layout->layout.ranges.end() ? 0 : static_cast<int64_t>(it->second.size());
}

int ew_layout_segments(const ew_layout* layout, int rank, ew_segment* out, int64_t cap) {
  if (layout == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL layout");
  const auto segs = elaskit::b200::shard_segments(layout->layout, rank);
  if (cap < static_cast<int64_t>(segs.size()))
    return set_error(EW_ERR_CAPACITY, "segment buffer too small");
  for (std::size_t i = 0; i < segs.size(); ++i)
    out[i] = ew_segment{segs[i].global_lo, segs[i].length, segs[i].local_off};
  return EW_OK;
}

int ew_layout_validate(const ew_layout* layout) {
  return guarded([&]() -> int {
    if (layout == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL layout");
    layout->layout.validate();
    return EW_OK;
  });
}

int ew_layout_owner_of(const ew_layout* layout, int64_t byte) {
  return layout ? layout->layout.owner_of(byte) : -1;
}

int ew_integrity_check(const int* ring_members, int n_ring, const ew_layout* layout,
                       const int* failed, int n_failed, int* recoverable, int* missing_ranks,
                       int missing_cap, int* n_missing) {
  return guarded([&]() -> int {
    if (layout == nullptr || recoverable == nullptr || n_ring < 0 || n_failed < 0)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_integrity_check: bad arguments");
    const auto rep =
        elaskit::integrity_check(to_ring(ring_members, n_ring), layout->layout, to_set(failed, n_failed));
    *recoverable = rep.recoverable ? 1 : 0;
    int k = 0;
    for (const auto& kv : rep.missing) {
      if (k < missing_cap && missing_ranks) missing_ranks[k] = kv.first;
      ++k;
    }
    if (n_missing) *n_missing = k;
    return k > missing_cap ? set_error(EW_ERR_CAPACITY, "missing-rank buffer too small") : EW_OK;
  });
}

int ew_overlap_matrix(const ew_layout* src, const ew_layout* dst, const int* failed,
                      int n_failed, const int* ring_members, int n_ring, ew_plan** out) {
  return guarded([&]() -> int {
    if (src == nullptr || dst == nullptr || out == nullptr || n_failed < 0 || n_ring < 0)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_overlap_matrix: bad arguments");
    *out = nullptr;
    const elaskit::SnapshotRing ring = to_ring(ring_members, n_ring);
    auto* p = new ew_plan{elaskit::overlap_matrix(src->layout, dst->layout,
                                                  to_set(failed, n_failed),
                                                  n_ring > 0 ? &ring : nullptr)};
    *out = p;
    return EW_OK;
  });
}

void ew_plan_free(ew_plan* plan) { delete plan; }

int64_t ew_plan_num_entries(const ew_plan* plan) {
  return plan ? static_cast<int64_t>(plan->plan.entries.size()) : -1;
}

int64_t ew_plan_total_bytes_moved(const ew_plan* plan) {
  return plan ? plan->plan.total_bytes_moved : -1;
}

int ew_plan_entries(const ew_plan* plan, ew_transfer_entry* out, int64_t cap) {
  if (plan == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL plan");
  if (cap < static_cast<int64_t>(plan->plan.entries.size()))
    return set_error(EW_ERR_CAPACITY, "entry buffer too small");
  std::size_t i = 0;
  for (const auto& e : plan->plan.entries)
    out[i++] = ew_transfer_entry{e.src_rank, e.dst_rank, e.iv.lo, e.iv.hi,
                                 e.medium == elaskit::Medium::D2D ? EW_MEDIUM_D2D
                                                                  : EW_MEDIUM_H2D_D2D,
                                 0};
  return EW_OK;
}

int ew_plan_to_json(const ew_plan* plan, char* buf, int64_t cap, int64_t* needed) {
  return guarded([&]() -> int {
    if (plan == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL plan");
    const std::string s = elaskit::plan_to_json(plan->plan).dump();
    if (needed) *needed = static_cast<int64_t>(s.size()) + 1;
    if (buf == nullptr || cap < static_cast<int64_t>(s.size()) + 1)
      return set_error(EW_ERR_CAPACITY, "json buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return EW_OK;
  });
}

int ew_reshard_copies(const ew_plan* plan, const ew_layout* src, const ew_layout* dst,
                      const int* failed, int n_failed, const int* ring_members, int n_ring,
                      int exec_rank, int push, ew_copy_desc* out, int64_t cap, int64_t* n_out) {
  return guarded([&]() -> int {
    if (plan == nullptr || src == nullptr || dst == nullptr || n_out == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_reshard_copies: bad arguments");
    const elaskit::SnapshotRing ring = to_ring(ring_members, n_ring);
    const auto copies = elaskit::b200::reshard_copies(
        plan->plan, src->layout, dst->layout, to_set(failed, n_failed),
        n_ring > 0 ? &ring : nullptr, exec_rank, push != 0);
    *n_out = static_cast<int64_t>(copies.size());
    const int64_t n = std::min<int64_t>(cap, static_cast<int64_t>(copies.size()));
    for (int64_t i = 0; i < n; ++i) {
      const auto& c = copies[static_cast<std::size_t>(i)];
      out[i] = ew_copy_desc{static_cast<int32_t>(c.src_role), c.src_rank,
                            static_cast<int32_t>(c.dst_role), c.dst_rank, c.src_off, c.dst_off,
                            c.bytes};
    }
    return static_cast<int64_t>(copies.size()) > cap
               ? set_error(EW_ERR_CAPACITY, "copy buffer too small")
               : EW_OK;
  });
}

int ew_inplace_schedule(const int64_t* layer_bytes, int n_layers, const ew_layout* src,
                        const ew_layout* dst, const int* failed, int n_failed,
                        int64_t stage_bytes, int64_t phase_bytes, int slack, ew_inplace** out) {
  return guarded([&]() -> int {
    if (out == nullptr || src == nullptr || dst == nullptr || n_layers < 0 ||
        (n_layers > 0 && layer_bytes == nullptr))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_inplace_schedule: bad arguments");
    *out = nullptr;
    auto* h = new ew_inplace{elaskit::b200::inplace_schedule(
        std::vector<int64_t>(layer_bytes, layer_bytes + n_layers), src->layout, dst->layout,
        to_set(failed, n_failed), stage_bytes, phase_bytes, slack)};
    *out = h;
    return EW_OK;
  });
}

int ew_inplace_info(const ew_inplace* s, int* descending, int* slack, int* ring,
                    int64_t* n_phases, int64_t* stage_alloc) {
  if (s == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL schedule");
  if (descending) *descending = s->s.descending ? 1 : 0;
  if (slack) *slack = s->s.slack;
  if (ring) *ring = s->s.ring;
  if (n_phases) *n_phases = static_cast<int64_t>(s->s.phases.size());
  if (stage_alloc) *stage_alloc = s->s.stage_alloc;
  return EW_OK;
}

int ew_inplace_phases(const ew_inplace* s, int64_t* out) {
  if (s == nullptr || (out == nullptr && !s->s.phases.empty()))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_inplace_phases: bad arguments");
  for (std::size_t j = 0; j < s->s.phases.size(); ++j) {
    out[2 * j] = s->s.phases[j].first;
    out[2 * j + 1] = s->s.phases[j].second;
  }
  return EW_OK;
}

int ew_inplace_ranges(const ew_inplace* s, int rank, int64_t* cut, int64_t* direct,
                      int64_t* staged) {
  if (s == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL schedule");
  const auto it = s->s.ranks.find(rank);
  if (it == s->s.ranks.end())
    return set_error(EW_ERR_INVALID_ARGUMENT, "rank " + std::to_string(rank) +
                                                  " is not in the target layout");
  const auto put = [](const std::vector<elaskit::b200::ByteRange>& v, int64_t* o) {
    if (o == nullptr) return;
    for (std::size_t j = 0; j < v.size(); ++j) {
      o[2 * j] = v[j].first;
      o[2 * j + 1] = v[j].second;
    }
  };
  put(it->second.cut, cut);
  put(it->second.direct, direct);
  put(it->second.staged, staged);
  return EW_OK;
}

void ew_inplace_free(ew_inplace* s) { delete s; }

int ew_reshard_microbatches(const int* old_per_slot_mbs, int n_old, int num_microbatches,
                            const int* survivors, int n_survivors, int* out_slots,
                            int* out_per_slot_mbs) {
  return guarded([&]() -> int {
    if (n_old < 0 || n_survivors < 0 || (n_survivors > 0 && (!out_slots || !out_per_slot_mbs)))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_reshard_microbatches: bad arguments");
    elaskit::MicrobatchAssignment old;
    old.per_slot_mbs.assign(old_per_slot_mbs, old_per_slot_mbs + n_old);
    old.slots.resize(static_cast<std::size_t>(n_old));
    for (int i = 0; i < n_old; ++i) old.slots[static_cast<std::size_t>(i)] = i;
    old.num_microbatches = num_microbatches;
    const auto next =
        elaskit::reshard_microbatches(old, std::vector<int>(survivors, survivors + n_survivors));
    for (std::size_t i = 0; i < next.slots.size(); ++i) {
      out_slots[i] = next.slots[i];
      out_per_slot_mbs[i] = next.per_slot_mbs[i];
    }
    return EW_OK;
  });
}

int ew_sample_reassignments(const int* old_slots, const int* old_mbs, int n_old,
                            const int* new_slots, const int* new_mbs, int n_new, int64_t* rows,
                            int64_t cap, int64_t* n_out) {
  return guarded([&]() -> int {
    if (n_old < 0 || n_new < 0 || n_out == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_sample_reassignments: bad arguments");
    elaskit::MicrobatchAssignment a, b;
    a.slots.assign(old_slots, old_slots + n_old);
    a.per_slot_mbs.assign(old_mbs, old_mbs + n_old);
    b.slots.assign(new_slots, new_slots + n_new);
    b.per_slot_mbs.assign(new_mbs, new_mbs + n_new);
    const auto r = elaskit::b200::sample_reassignments(a, b);
    *n_out = static_cast<int64_t>(r.size());
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n_out); ++i) {
      rows[3 * i] = r[static_cast<std::size_t>(i)].sample_id;
      rows[3 * i + 1] = r[static_cast<std::size_t>(i)].old_slot;
      rows[3 * i + 2] = r[static_cast<std::size_t>(i)].new_slot;
    }
    return *n_out > cap ? set_error(EW_ERR_CAPACITY, "row buffer too small") : EW_OK;
  });
}

int ew_plan_zero_migration(int kind, int dp_degree, const int64_t* layer_bytes, int n_layers,
                           int layer_idx, int dst_dp_degree, int64_t* rows, int64_t cap,
                           int64_t* n_out, int64_t* totals) {
  return guarded([&]() -> int {
    if (n_layers < 0 || n_out == nullptr || totals == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_plan_zero_migration: bad arguments");
    elaskit::ZeroLayout z;
    z.kind = kind ? elaskit::ZeroKind::Interleaved : elaskit::ZeroKind::Contiguous;
    z.dp_degree = dp_degree;
    z.layer_bytes.assign(layer_bytes, layer_bytes + n_layers);
    const auto p = elaskit::plan_zero_migration(layer_idx, z, dst_dp_degree);
    *n_out = static_cast<int64_t>(p.transfers.size());
    totals[0] = p.cross_bytes;
    totals[1] = p.intra_bytes;
    totals[2] = p.total_bytes;
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n_out); ++i) {
      const auto& t = p.transfers[static_cast<std::size_t>(i)];
      int64_t* row = rows + 6 * i;
      row[0] = t.src_rank;
      row[1] = t.dst_rank;
      row[2] = t.cross_stage ? 1 : 0;
      row[3] = t.iv.lo;
      row[4] = t.iv.hi;
      row[5] = t.round;
    }
    return *n_out > cap ? set_error(EW_ERR_CAPACITY, "row buffer too small") : EW_OK;
  });
}

int ew_plan_layer_migration(int layer, int src_stage, int dst_stage, int mode,
                            const ew_migration_context* ctx, ew_migration_schedule* out) {
  return guarded([&]() -> int {
    if (ctx == nullptr || out == nullptr || (mode != 0 && mode != 1))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_plan_layer_migration: bad arguments");
    elaskit::LayerMove mv;
    mv.layer = layer;
    mv.src_stage = src_stage;
    mv.dst_stage = dst_stage;
    elaskit::MigrationContext c;
    c.param_bytes = ctx->param_bytes;
    c.grad_bytes = ctx->grad_bytes;
    c.link_bw_bytes_per_s = ctx->link_bw_bytes_per_s;
    c.microbatch_slot_s = ctx->microbatch_slot_s;
    c.num_microbatches = ctx->num_microbatches;
    c.target_headroom_bytes = ctx->target_headroom_bytes;
    c.fixed_overhead_s = ctx->fixed_overhead_s;
    const auto s = elaskit::plan_layer_migration(
        mv, mode ? elaskit::MigrationMode::NonBlocking : elaskit::MigrationMode::Blocking, c);
    *out = ew_migration_schedule{};
    out->mode = s.mode == elaskit::MigrationMode::NonBlocking ? 1 : 0;
    out->shadow_microbatches = s.shadow_microbatches;
    out->n_transfers = static_cast<int32_t>(std::min<std::size_t>(2, s.transfers.size()));
    for (int i = 0; i < out->n_transfers; ++i) {
      const auto& t = s.transfers[static_cast<std::size_t>(i)];
      out->transfers[i] = {t.what == "payback_grad" ? 1 : 0, t.start_s, t.end_s, t.bytes};
    }
    out->payback_bytes = s.payback_bytes;
    out->stall_s = s.stall_s;
    out->total_time_s = s.total_time_s;
    return EW_OK;
  });
}

int ew_weighted_grad_average(const double* weights, const double* grads, int n, int64_t dim,
                             double* out) {
  return guarded([&]() -> int {
    if (n < 0 || dim < 0 || (n > 0 && (!weights || !grads)) || (dim > 0 && n > 0 && !out))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_weighted_grad_average: bad arguments");
    std::vector<std::pair<double, std::vector<double>>> c;
    c.reserve(static_cast<std::size_t>(n));
    for (int j = 0; j < n; ++j)
      c.push_back({weights[j], std::vector<double>(grads + j * dim, grads + (j + 1) * dim)});
    const auto acc = elaskit::weighted_grad_average(c);
    std::memcpy(out, acc.data(), acc.size() * sizeof(double));
    return EW_OK;
  });
}

int ew_philox4x64(const uint64_t counter[4], const uint64_t key[2], uint64_t out[4]) {
  if (!counter || !key || !out) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL argument");
  const auto w = elaskit::philox4x64({counter[0], counter[1], counter[2], counter[3]},
                                     {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = w[static_cast<std::size_t>(i)];
  return EW_OK;
}

int ew_draw(uint64_t seed, uint64_t sample_id, uint32_t layer_id, uint32_t op_index, int n,
            double* out) {
  return guarded([&]() -> int {
    const auto u = elaskit::draw({seed, sample_id, layer_id, op_index}, n);
    if (out == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL out");
    std::memcpy(out, u.data(), u.size() * sizeof(double));
    return EW_OK;
  });
}

int ew_plan_edit(int n_groups, const char* const* ids, const int* topo, const int* n_members,
                 const int* members, int event_kind, const int* targets, int n_targets,
                 const int* pool_links, int n_pool, int* add_links, int add_cap, int* n_add,
                 int* remove_links, int remove_cap, int* n_remove, int* touched_groups,
                 int* n_touched) {
  return guarded([&]() -> int {
    if (n_groups < 0 || event_kind < 0 || event_kind > 3 || n_targets < 0 || n_pool < 0)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_plan_edit: bad arguments");
    std::vector<elaskit::CommGroup> groups;
    int64_t k = 0;
    for (int g = 0; g < n_groups; ++g) {
      elaskit::CommGroup cg;
      cg.id = ids ? ids[g] : std::to_string(g);
      cg.topo = topo[g] ? elaskit::GroupTopology::Ring : elaskit::GroupTopology::Mesh;
      for (int m = 0; m < n_members[g]; ++m) cg.members.push_back(members[k++]);
      groups.push_back(cg);
    }
    elaskit::ElasticEvent ev;
    ev.kind = static_cast<elaskit::EventKind>(event_kind);
    ev.targets.assign(targets, targets + n_targets);
    std::set<elaskit::Link> pool;
    for (int i = 0; i < n_pool; ++i) pool.insert(elaskit::make_link(pool_links[2 * i], pool_links[2 * i + 1]));
    const auto plan = elaskit::plan_edit(groups, ev, pool);
    int i = 0;
    for (const auto& l : plan.links_to_add) {
      if (i < add_cap) {
        add_links[2 * i] = l.first;
        add_links[2 * i + 1] = l.second;
      }
      ++i;
    }
    *n_add = i;
    i = 0;
    for (const auto& l : plan.links_to_remove) {
      if (i < remove_cap) {
        remove_links[2 * i] = l.first;
        remove_links[2 * i + 1] = l.second;
      }
      ++i;
    }
    *n_remove = i;
    i = 0;
    for (int g = 0; g < n_groups; ++g)
      if (plan.groups_touched.contains(groups[static_cast<std::size_t>(g)].id))
        touched_groups[i++] = g;
    *n_touched = i;
    if (*n_add > add_cap || *n_remove > remove_cap)
      return set_error(EW_ERR_CAPACITY, "link buffers too small");
    return EW_OK;
  });
}

}  // extern "C"
