// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the *reference* elaskit library, compiled together
// with the unmodified reference sources under /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libelaskit_ref.so.  Tests and bench.py's
// CPU baseline call the reference's own implementation through it (ctypes)
// to pin the B200 build's planners and the oracle restatement against the
// reference itself.  Status codes follow include/ew_api.h.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "elaskit/communicator.hpp"
#include "elaskit/dataflow.hpp"
#include "elaskit/migration.hpp"
#include "elaskit/param_fabric.hpp"
#include "elaskit/rng.hpp"

using namespace elaskit;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const CoverageMismatch& e) {
    g_err = e.what();
    return 2;
  } catch (const MissingBackup& e) {
    g_err = e.what();
    return 3;
  } catch (const NoSurvivors& e) {
    g_err = e.what();
    return 4;
  } catch (const DimensionMismatch& e) {
    g_err = e.what();
    return 5;
  } catch (const MismatchedDpDegree& e) {
    g_err = e.what();
    return 6;
  } catch (const DisconnectedGroup& e) {
    g_err = e.what();
    return 7;
  } catch (const InsufficientTargetMemory& e) {
    g_err = e.what();
    return 13;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 8;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 12;
  }
}

PartitionLayout make_layout(const int* ranks, const int* counts, int n_ranks,
                            const int64_t* ivs, int64_t total) {
  PartitionLayout l;
  l.total_bytes = total;
  int64_t k = 0;
  for (int i = 0; i < n_ranks; ++i) {
    auto& v = l.ranges[ranks[i]];
    for (int c = 0; c < counts[i]; ++c, ++k) v.push_back({ivs[2 * k], ivs[2 * k + 1]});
  }
  return l;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// overlap_matrix (param_fabric.cpp:82-121).  Entries as int64 rows
// {src, dst, lo, hi, medium}; returns status, *n_entries, *total_moved.
int ref_overlap_matrix(const int* s_ranks, const int* s_counts, int s_n, const int64_t* s_ivs,
                       const int* d_ranks, const int* d_counts, int d_n, const int64_t* d_ivs,
                       int64_t total, const int* failed, int n_failed, const int* ring,
                       int n_ring, int64_t* out, int64_t cap, int64_t* n_entries,
                       int64_t* total_moved, double* seconds) {
  return guarded([&]() -> int {
    const PartitionLayout src = make_layout(s_ranks, s_counts, s_n, s_ivs, total);
    const PartitionLayout dst = make_layout(d_ranks, d_counts, d_n, d_ivs, total);
    std::set<int> f(failed, failed + n_failed);
    SnapshotRing r;
    r.members.assign(ring, ring + n_ring);
    const auto t0 = std::chrono::steady_clock::now();
    const TransferPlan p = overlap_matrix(src, dst, f, n_ring > 0 ? &r : nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    *n_entries = static_cast<int64_t>(p.entries.size());
    *total_moved = p.total_bytes_moved;
    if (cap < *n_entries) return 9;
    for (std::size_t i = 0; i < p.entries.size(); ++i) {
      const TransferEntry& e = p.entries[i];
      out[5 * i + 0] = e.src_rank;
      out[5 * i + 1] = e.dst_rank;
      out[5 * i + 2] = e.iv.lo;
      out[5 * i + 3] = e.iv.hi;
      out[5 * i + 4] = e.medium == Medium::D2D ? 0 : 1;
    }
    return 0;
  });
}

int ref_plan_to_json(const int* s_ranks, const int* s_counts, int s_n, const int64_t* s_ivs,
                     const int* d_ranks, const int* d_counts, int d_n, const int64_t* d_ivs,
                     int64_t total, const int* failed, int n_failed, const int* ring, int n_ring,
                     char* buf, int64_t cap) {
  return guarded([&]() -> int {
    const PartitionLayout src = make_layout(s_ranks, s_counts, s_n, s_ivs, total);
    const PartitionLayout dst = make_layout(d_ranks, d_counts, d_n, d_ivs, total);
    std::set<int> f(failed, failed + n_failed);
    SnapshotRing r;
    r.members.assign(ring, ring + n_ring);
    const std::string s = plan_to_json(overlap_matrix(src, dst, f, n_ring > 0 ? &r : nullptr)).dump();
    if (cap < static_cast<int64_t>(s.size()) + 1) return 9;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
  });
}

int ref_integrity_check(const int* ring, int n_ring, const int* ranks, const int* counts, int n,
                        const int64_t* ivs, int64_t total, const int* failed, int n_failed,
                        int* recoverable, int* missing, int* n_missing) {
  return guarded([&]() -> int {
    SnapshotRing r;
    r.members.assign(ring, ring + n_ring);
    const auto rep = integrity_check(r, make_layout(ranks, counts, n, ivs, total),
                                     std::set<int>(failed, failed + n_failed));
    *recoverable = rep.recoverable;
    int k = 0;
    for (const auto& kv : rep.missing) missing[k++] = kv.first;
    *n_missing = k;
    return 0;
  });
}

// ZeroLayout::shard (migration.cpp:73-77) for the interleaved composition.
int ref_zero_shard(const int64_t* layer_bytes, int n_layers, int dp, int layer, int rank,
                   int64_t* lo, int64_t* hi, int64_t* layer_offset) {
  return guarded([&]() -> int {
    ZeroLayout z;
    z.kind = ZeroKind::Interleaved;
    z.dp_degree = dp;
    z.layer_bytes.assign(layer_bytes, layer_bytes + n_layers);
    const ByteInterval s = z.shard(layer, rank);
    *lo = s.lo;
    *hi = s.hi;
    *layer_offset = z.layer_offset(layer);
    return 0;
  });
}

// plan_zero_migration (migration.cpp:87-154); rows {src,dst,cross,lo,hi,round}.
int ref_plan_zero_migration(int kind, int dp, const int64_t* layer_bytes, int n_layers,
                            int layer, int dst_dp, int64_t* out, int64_t cap, int64_t* n_out,
                            int64_t* totals) {
  return guarded([&]() -> int {
    ZeroLayout z;
    z.kind = kind ? ZeroKind::Interleaved : ZeroKind::Contiguous;
    z.dp_degree = dp;
    z.layer_bytes.assign(layer_bytes, layer_bytes + n_layers);
    const auto p = plan_zero_migration(layer, z, dst_dp);
    *n_out = static_cast<int64_t>(p.transfers.size());
    totals[0] = p.cross_bytes;
    totals[1] = p.intra_bytes;
    totals[2] = p.total_bytes;
    if (cap < *n_out) return 9;
    for (std::size_t i = 0; i < p.transfers.size(); ++i) {
      const auto& t = p.transfers[i];
      int64_t* row = out + 6 * i;
      row[0] = t.src_rank;
      row[1] = t.dst_rank;
      row[2] = t.cross_stage;
      row[3] = t.iv.lo;
      row[4] = t.iv.hi;
      row[5] = t.round;
    }
    return 0;
  });
}

// plan_layer_migration (migration.cpp:9-61).  ictx {param_bytes, grad_bytes,
// num_microbatches, target_headroom}, dctx {link_bw, slot_s, fixed_overhead};
// iout {mode, shadow_mbs, n_transfers, payback_bytes, what0, bytes0, what1,
// bytes1}, dout {stall, total, start0, end0, start1, end1}.
int ref_plan_layer_migration(int layer, int src, int dst, int mode, const int64_t* ictx,
                             const double* dctx, int64_t* iout, double* dout) {
  return guarded([&]() -> int {
    LayerMove mv;
    mv.layer = layer;
    mv.src_stage = src;
    mv.dst_stage = dst;
    MigrationContext c;
    c.param_bytes = ictx[0];
    c.grad_bytes = ictx[1];
    c.num_microbatches = static_cast<int>(ictx[2]);
    c.target_headroom_bytes = ictx[3];
    c.link_bw_bytes_per_s = dctx[0];
    c.microbatch_slot_s = dctx[1];
    c.fixed_overhead_s = dctx[2];
    const auto s = plan_layer_migration(mv, mode ? MigrationMode::NonBlocking : MigrationMode::Blocking, c);
    iout[0] = s.mode == MigrationMode::NonBlocking ? 1 : 0;
    iout[1] = s.shadow_microbatches;
    iout[2] = static_cast<int64_t>(s.transfers.size());
    iout[3] = s.payback_bytes;
    dout[0] = s.stall_s;
    dout[1] = s.total_time_s;
    for (std::size_t i = 0; i < s.transfers.size() && i < 2; ++i) {
      iout[4 + 2 * i] = s.transfers[i].what == "payback_grad" ? 1 : 0;
      iout[5 + 2 * i] = s.transfers[i].bytes;
      dout[2 + 2 * i] = s.transfers[i].start_s;
      dout[3 + 2 * i] = s.transfers[i].end_s;
    }
    return 0;
  });
}

int ref_philox4x64(const uint64_t* counter, const uint64_t* key, uint64_t* out) {
  const auto w = philox4x64({counter[0], counter[1], counter[2], counter[3]}, {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = w[i];
  return 0;
}

int ref_draw(uint64_t seed, uint64_t sample, uint32_t layer, uint32_t op, int n, double* out) {
  return guarded([&]() -> int {
    const auto v = draw({seed, sample, layer, op}, n);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    return 0;
  });
}

// Reference draw() over many samples, as the CPU baseline of the mask kernel:
// out bits use the sim.cpp:926-928 rule (bit set = kept).
int ref_dropout_mask(uint64_t seed, uint64_t sample_lo, int64_t n_samples, uint32_t layer,
                     uint32_t op, int n_elems, double keep, uint32_t* bits) {
  return guarded([&]() -> int {
    const int64_t wpr = (n_elems + 31) / 32;
    for (int64_t s = 0; s < n_samples; ++s) {
      const auto u = draw({seed, sample_lo + static_cast<uint64_t>(s), layer, op}, n_elems);
      uint32_t* row = bits + s * wpr;
      std::memset(row, 0, static_cast<std::size_t>(wpr) * 4);
      for (int k = 0; k < n_elems; ++k)
        if (!(u[k] < keep)) row[k / 32] |= 1u << (k % 32);
    }
    return 0;
  });
}

int ref_weighted_grad_average(const double* w, const double* g, int n, int64_t dim,
                              double* out) {
  return guarded([&]() -> int {
    std::vector<std::pair<double, std::vector<double>>> c;
    for (int j = 0; j < n; ++j) c.push_back({w[j], std::vector<double>(g + j * dim, g + (j + 1) * dim)});
    const auto acc = weighted_grad_average(c);
    std::memcpy(out, acc.data(), acc.size() * sizeof(double));
    return 0;
  });
}

int ref_reshard_microbatches(const int* old_mbs, int n_old, int num_mb, const int* survivors,
                             int n_surv, int* out_slots, int* out_mbs) {
  return guarded([&]() -> int {
    MicrobatchAssignment a;
    a.per_slot_mbs.assign(old_mbs, old_mbs + n_old);
    for (int i = 0; i < n_old; ++i) a.slots.push_back(i);
    a.num_microbatches = num_mb;
    const auto b = reshard_microbatches(a, std::vector<int>(survivors, survivors + n_surv));
    for (std::size_t i = 0; i < b.slots.size(); ++i) {
      out_slots[i] = b.slots[i];
      out_mbs[i] = b.per_slot_mbs[i];
    }
    return 0;
  });
}

int ref_plan_edit(int n_groups, const char* const* ids, const int* topo, const int* n_members,
                  const int* members, int kind, const int* targets, int n_targets,
                  const int* pool, int n_pool, int* add, int* n_add, int* rem, int* n_rem,
                  int* touched, int* n_touched) {
  return guarded([&]() -> int {
    std::vector<CommGroup> gs;
    int64_t k = 0;
    for (int g = 0; g < n_groups; ++g) {
      CommGroup cg;
      cg.id = ids[g];
      cg.topo = topo[g] ? GroupTopology::Ring : GroupTopology::Mesh;
      for (int m = 0; m < n_members[g]; ++m) cg.members.push_back(members[k++]);
      gs.push_back(cg);
    }
    ElasticEvent ev;
    ev.kind = static_cast<EventKind>(kind);
    ev.targets.assign(targets, targets + n_targets);
    std::set<Link> p;
    for (int i = 0; i < n_pool; ++i) p.insert(make_link(pool[2 * i], pool[2 * i + 1]));
    const auto plan = plan_edit(gs, ev, p);
    int i = 0;
    for (const auto& l : plan.links_to_add) {
      add[2 * i] = l.first;
      add[2 * i + 1] = l.second;
      ++i;
    }
    *n_add = i;
    i = 0;
    for (const auto& l : plan.links_to_remove) {
      rem[2 * i] = l.first;
      rem[2 * i + 1] = l.second;
      ++i;
    }
    *n_rem = i;
    i = 0;
    for (int g = 0; g < n_groups; ++g)
      if (plan.groups_touched.contains(gs[g].id)) touched[i++] = g;
    *n_touched = i;
    return 0;
  });
}

}  // extern "C"
