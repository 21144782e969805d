// C ABI over the multi-process recovery runtime (include/elaskit/recovery.hpp):
// stores, channels, peer mappings, reshard executors, prepared recoveries,
// the DP group and the in-place executor, for foreign callers (the Python
// binding, cgo, JNI).  Opaque handles own their C++ objects; nothing throws
// across the boundary (host/guarded.hpp).
#include <cstring>
#include <memory>
#include <string>

#include "elaskit/recovery.hpp"
#include "host/guarded.hpp"

using elaskit::b200::Channel;
using elaskit::b200::DpGroup;
using elaskit::b200::InPlaceExecutor;
using elaskit::b200::MttrEvent;
using elaskit::b200::PeerBuffers;
using elaskit::b200::PreparedRecovery;
using elaskit::b200::ReshardExecutor;
using elaskit::b200::ReshardPlan;
using elaskit::b200::Store;
using ew::guarded;
using ew::set_error;

struct ew_layout {
  elaskit::PartitionLayout layout;
};
struct ew_store {
  std::unique_ptr<Store> s;
};
struct ew_channel {
  std::unique_ptr<Channel> c;
};
struct ew_peers {
  PeerBuffers p;
};
struct ew_reshard {
  std::unique_ptr<ReshardExecutor> x;
};
struct ew_prepared {
  std::unique_ptr<PreparedRecovery> p;
};
struct ew_dp_group {
  std::unique_ptr<DpGroup> g;
};
struct ew_detector {
  std::unique_ptr<elaskit::b200::FailureDetector> d;
};
struct ew_inplace_exec {
  std::unique_ptr<InPlaceExecutor> x;
};
struct ew_replay_replica {
  std::unique_ptr<elaskit::b200::ReplayReplica> r;
};
struct ew_ring_replica {
  std::unique_ptr<elaskit::b200::RingReplica> r;
};
struct ew_peer_reduce {
  std::unique_ptr<elaskit::b200::PeerReduce> r;
};
struct ew_host_images {
  std::unique_ptr<elaskit::b200::HostImages> h;
};
struct ew_layer_migration {
  std::unique_ptr<elaskit::b200::LayerMigration> m;
};

namespace {

void to_c(const MttrEvent& ev, ew_mttr_event* out) {
  if (out == nullptr) return;
  std::memset(out, 0, sizeof(*out));
  out->step = ev.step;
  out->verified = ev.verified ? 1 : 0;
  out->t_event_s = ev.t_event_s;
  std::strncpy(out->kind, ev.kind.c_str(), sizeof(out->kind) - 1);
  out->detect_s = ev.detect_s;
  out->comm_repair_s = ev.comm_repair_s;
  out->remap_s = ev.remap_s;
  out->migration_stall_s = ev.migration_stall_s;
  out->other_s = ev.other_s;
  out->lost_work_s = ev.lost_work_s;
  auto ph = [&](const char* k) {
    const auto it = ev.phases.find(k);
    return it == ev.phases.end() ? -1.0 : it->second;
  };
  out->plan_edit_s = ph("plan_edit_s");
  out->comm_acquire_s = ph("comm_acquire_s");
  out->first_collective_s = ph("first_collective_s");
  out->comm_prepared = ph("comm_prepared");
  out->plan_s = ph("plan_s");
  out->map_bind_s = ph("map_bind_s");
  out->copy_s = ph("copy_s");
  out->barrier_verify_s = ph("barrier_verify_s");
  out->verdict_exchange_s = ph("verdict_exchange_s");
  out->launch_to_verdict_s = ph("launch_to_verdict_s");
  out->mismatched_block_words = ph("mismatched_block_words");
  out->barrier_timeouts = ph("barrier_timeouts");
  out->premapped = ph("premapped");
  out->sums_s = ph("sums_s");
  out->bind_s = ph("bind_s");
  out->prepared = ph("prepared");
  out->stale_snapshots = ph("stale_snapshots");
}

MttrEvent from_c(const ew_mttr_event& e) {
  MttrEvent ev;
  ev.step = e.step;
  ev.verified = e.verified != 0;
  ev.t_event_s = e.t_event_s;
  ev.kind = std::string(e.kind, strnlen(e.kind, sizeof(e.kind)));
  ev.detect_s = e.detect_s;
  ev.comm_repair_s = e.comm_repair_s;
  ev.remap_s = e.remap_s;
  ev.migration_stall_s = e.migration_stall_s;
  ev.other_s = e.other_s;
  ev.lost_work_s = e.lost_work_s;
  return ev;
}

int copy_out(const std::string& s, char* buf, int64_t cap) {
  if (buf == nullptr || cap < 1) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (static_cast<int64_t>(s.size()) + 1 > cap) return set_error(EW_ERR_CAPACITY, "buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return EW_OK;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ stores

int ew_store_tcp(const char* host, int port, int is_server, double timeout_s, ew_store** out) {
  return guarded([&]() -> int {
    if (host == nullptr || out == nullptr || port <= 0 || port > 65535)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_store_tcp: bad arguments");
    *out = new ew_store{elaskit::b200::tcp_store(host, port, is_server != 0, timeout_s)};
    return EW_OK;
  });
}

int ew_store_callbacks(ew_store_set_fn set, ew_store_get_fn get, ew_store_erase_fn erase,
                       void* ctx, ew_store** out) {
  return guarded([&]() -> int {
    if (set == nullptr || get == nullptr || out == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_store_callbacks: bad arguments");
    auto s = [set, ctx](const std::string& k, const std::string& v) {
      if (set(ctx, k.data(), static_cast<int64_t>(k.size()), v.data(),
              static_cast<int64_t>(v.size())) != 0)
        throw std::runtime_error("store set callback failed for key " + k);
    };
    auto g = [get, ctx](const std::string& k) {
      std::string v(256, '\0');
      for (int attempt = 0; attempt < 2; ++attempt) {
        int64_t n = 0;
        const int st = get(ctx, k.data(), static_cast<int64_t>(k.size()), v.data(),
                           static_cast<int64_t>(v.size()), &n);
        if (st == 0 && n <= static_cast<int64_t>(v.size())) {
          v.resize(static_cast<std::size_t>(n));
          return v;
        }
        if (st != 0 && st != EW_ERR_CAPACITY)
          throw std::runtime_error("store get callback failed for key " + k);
        v.assign(static_cast<std::size_t>(n), '\0');  // retry with the size it asked for
      }
      throw std::runtime_error("store get callback: size changed between calls for " + k);
    };
    std::function<void(const std::string&)> e;
    if (erase != nullptr)
      e = [erase, ctx](const std::string& k) {
        if (erase(ctx, k.data(), static_cast<int64_t>(k.size())) != 0)
          throw std::runtime_error("store erase callback failed for key " + k);
      };
    *out = new ew_store{elaskit::b200::callback_store(s, g, e)};
    return EW_OK;
  });
}

int ew_store_set(ew_store* st, const char* key, const void* val, int64_t len) {
  return guarded([&]() -> int {
    if (st == nullptr || key == nullptr || (len > 0 && val == nullptr) || len < 0)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_store_set: bad arguments");
    st->s->set(key, std::string(static_cast<const char*>(val), static_cast<std::size_t>(len)));
    return EW_OK;
  });
}

int ew_store_get(ew_store* st, const char* key, void* buf, int64_t cap, int64_t* len) {
  return guarded([&]() -> int {
    if (st == nullptr || key == nullptr || len == nullptr || (cap > 0 && buf == nullptr))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_store_get: bad arguments");
    const std::string v = st->s->get(key);
    *len = static_cast<int64_t>(v.size());
    if (*len > cap) return set_error(EW_ERR_CAPACITY, "ew_store_get: buffer too small");
    std::memcpy(buf, v.data(), v.size());
    return EW_OK;
  });
}

void ew_store_free(ew_store* st) { delete st; }

int ew_channel_create(ew_store* st, const char* name, const int* members, int n, int me,
                      ew_channel** out) {
  return guarded([&]() -> int {
    if (st == nullptr || name == nullptr || out == nullptr || n < 1 || members == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_channel_create: bad arguments");
    *out = new ew_channel{std::make_unique<Channel>(*st->s, name,
                                                    std::vector<int>(members, members + n), me)};
    return EW_OK;
  });
}

int ew_channel_barrier(ew_channel* ch) {
  return guarded([&]() -> int {
    if (ch == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL channel");
    ch->c->barrier();
    return EW_OK;
  });
}

int ew_channel_sum(ew_channel* ch, int64_t mine, int64_t* total) {
  return guarded([&]() -> int {
    if (ch == nullptr || total == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    *total = ch->c->sum(mine);
    return EW_OK;
  });
}

void ew_channel_free(ew_channel* ch) { delete ch; }

// ------------------------------------------------------------------- MTTR

int ew_mttr_csv_header(char* buf, int64_t cap) {
  return copy_out(elaskit::b200::mttr_csv_header(), buf, cap);
}

int ew_mttr_csv_row(const ew_mttr_event* ev, int index, char* buf, int64_t cap) {
  if (ev == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL event");
  return copy_out(elaskit::b200::mttr_csv_row(index, from_c(*ev)), buf, cap);
}

// ------------------------------------------------------------ peer buffers

int ew_peers_create(ew_peers** out) {
  if (out == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  *out = new ew_peers();
  return EW_OK;
}

int ew_peers_exchange(ew_peers* p, ew_channel* ch, const int* keys, void* const* ptrs, int n) {
  return guarded([&]() -> int {
    if (p == nullptr || ch == nullptr || n < 0 || (n > 0 && (!keys || !ptrs)))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_peers_exchange: bad arguments");
    std::map<int, void*> mine;
    for (int i = 0; i < n; ++i) mine[keys[i]] = ptrs[i];
    p->p.exchange(*ch->c, mine);
    return EW_OK;
  });
}

int ew_peers_put(ew_peers* p, int key, int member, void* ptr) {
  if (p == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  p->p.put(key, member, ptr);
  return EW_OK;
}

int ew_peers_get(const ew_peers* p, int key, int member, void** ptr) {
  if (p == nullptr || ptr == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  *ptr = p->p.get(key, member);
  return EW_OK;
}

void ew_peers_free(ew_peers* p) { delete p; }

// ---------------------------------------------------------------- reshard

int ew_reshard_create(const ew_layout* src, const ew_layout* dst, const int* failed, int n_failed,
                      const int* ring, int n_ring, int me, int push, int64_t block_bytes,
                      ew_reshard** out) {
  return guarded([&]() -> int {
    if (src == nullptr || dst == nullptr || out == nullptr || n_failed < 0 || n_ring < 0 ||
        (n_failed && !failed) || (n_ring && !ring))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_reshard_create: bad arguments");
    const ReshardPlan rp = ReshardPlan::from_layouts(
        src->layout, dst->layout, std::set<int>(failed, failed + n_failed),
        std::vector<int>(ring, ring + n_ring));
    *out = new ew_reshard{std::make_unique<ReshardExecutor>(rp, me, push != 0, block_bytes)};
    return EW_OK;
  });
}

int ew_reshard_bind(ew_reshard* r, const ew_peers* peers, int verify) {
  return guarded([&]() -> int {
    if (r == nullptr || peers == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    r->x->bind(peers->p, verify != 0);
    return EW_OK;
  });
}

int ew_reshard_launch(const ew_reshard* r, uint64_t* block_sums, const int* abort_flag,
                      int n_ctas, int remote_ctas, ew_stream_t stream) {
  return guarded([&]() -> int {
    if (r == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    r->x->launch(stream, block_sums, abort_flag, n_ctas, remote_ctas);
    return EW_OK;
  });
}

void ew_reshard_free(ew_reshard* r) { delete r; }

// ------------------------------------------------------- prepared recovery

int ew_prepared_create(ew_channel* ch, const int64_t* layer_bytes, int n_layers, void* old_buf,
                       const uint64_t* old_rows, void* replica, const uint64_t* replica_rows,
                       void* new_buf, int64_t new_capacity, int64_t block_bytes,
                       double barrier_timeout_s, int flags, ew_prepared** out) {
  return guarded([&]() -> int {
    if (ch == nullptr || layer_bytes == nullptr || n_layers < 1 || out == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_prepared_create: bad arguments");
    elaskit::b200::PreparedOptions opt;
    opt.block_bytes = block_bytes;
    opt.barrier_timeout_s = barrier_timeout_s;
    opt.local_replicas = (flags & 1) != 0;
    *out = new ew_prepared{std::make_unique<PreparedRecovery>(
        *ch->c, std::vector<int64_t>(layer_bytes, layer_bytes + n_layers), old_buf, old_rows,
        replica, replica_rows, new_buf, new_capacity, opt)};
    return EW_OK;
  });
}

int ew_prepared_recover(ew_prepared* p, int departed, ew_stream_t stream, ew_mttr_event* ev,
                        int* verified) {
  return guarded([&]() -> int {
    if (p == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    MttrEvent e;
    const bool ok = p->p->recover(departed, stream, &e);
    if (verified) *verified = ok ? 1 : 0;
    to_c(e, ev);
    return EW_OK;
  });
}

int ew_prepared_new(const ew_prepared* p, int departed, void** ptr, int64_t* bytes) {
  return guarded([&]() -> int {
    if (p == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    if (ptr) *ptr = p->p->new_buf();
    if (bytes) *bytes = p->p->new_bytes(departed);
    return EW_OK;
  });
}

void ew_prepared_free(ew_prepared* p) { delete p; }

// ---------------------------------------------------------------- DP group

int ew_dp_group_create(ew_channel* ch, const int64_t* layer_bytes, int n_layers, ew_comm* comm,
                       int per_slot_mbs, int num_microbatches, int64_t block_bytes,
                       int prepare_comms, ew_dp_group** out) {
  return guarded([&]() -> int {
    if (ch == nullptr || layer_bytes == nullptr || n_layers < 1 || out == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_dp_group_create: bad arguments");
    elaskit::b200::DpGroupOptions opt;
    opt.per_slot_mbs = per_slot_mbs;
    opt.num_microbatches = num_microbatches;
    opt.block_bytes = block_bytes;
    opt.prepare_comms = (prepare_comms & 1) != 0;
    opt.share_comm_resources = (prepare_comms & 2) != 0;
    *out = new ew_dp_group{std::make_unique<DpGroup>(
        *ch->c, std::vector<int64_t>(layer_bytes, layer_bytes + n_layers), comm, opt)};
    return EW_OK;
  });
}

int ew_dp_group_create_joiner(ew_store* store, const char* group_name, const int64_t* layer_bytes,
                              int n_layers, const int* members, int n_members, int me,
                              int per_slot_mbs, int num_microbatches, int64_t block_bytes,
                              ew_dp_group** out) {
  return guarded([&]() -> int {
    if (store == nullptr || group_name == nullptr || layer_bytes == nullptr || n_layers < 1 ||
        members == nullptr || n_members < 1 || out == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_dp_group_create_joiner: bad arguments");
    elaskit::b200::DpGroupOptions opt;
    opt.per_slot_mbs = per_slot_mbs;
    opt.num_microbatches = num_microbatches;
    opt.block_bytes = block_bytes;
    opt.prepare_comms = false;
    *out = new ew_dp_group{std::make_unique<DpGroup>(
        *store->s, std::string(group_name), std::vector<int64_t>(layer_bytes, layer_bytes + n_layers),
        std::vector<int>(members, members + n_members), me, opt)};
    return EW_OK;
  });
}

int ew_dp_group_prepare_join(ew_dp_group* g, const int* joiners, int n) {
  return guarded([&]() -> int {
    if (g == nullptr || joiners == nullptr || n < 1)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_dp_group_prepare_join: bad arguments");
    g->g->prepare_join(std::vector<int>(joiners, joiners + n));
    return EW_OK;
  });
}

int ew_dp_group_premap(ew_dp_group* g, void* old_buf, void* replica, const uint64_t* old_rows,
                       const uint64_t* replica_rows) {
  return guarded([&]() -> int {
    if (g == nullptr || old_buf == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_dp_group_premap: bad arguments");
    elaskit::b200::RankBuffers b;
    b.old_buf = old_buf;
    b.replica = replica;
    g->g->premap(b, old_rows, replica_rows);
    return EW_OK;
  });
}

int ew_dp_group_prepare_move(ew_dp_group* g, int kind, const int* targets, int n, void* new_buf) {
  return guarded([&]() -> int {
    if (g == nullptr || targets == nullptr || n < 1 || kind < 0 || kind > 3)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_dp_group_prepare_move: bad arguments");
    g->g->prepare_move(static_cast<elaskit::EventKind>(kind),
                       std::vector<int>(targets, targets + n), new_buf);
    return EW_OK;
  });
}

int ew_dp_group_set_snapshot_step(ew_dp_group* g, int64_t step) {
  if (g == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL group");
  g->g->set_snapshot_step(step);
  return EW_OK;
}

int ew_dp_group_attach(ew_dp_group* g, ew_prepared* p) {
  if (g == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  g->g->attach(p ? p->p.get() : nullptr);
  return EW_OK;
}

int ew_dp_group_prepare(ew_dp_group* g) {
  return guarded([&]() -> int {
    if (g == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    g->g->prepare();
    return EW_OK;
  });
}

int ew_dp_group_prepare_sets(ew_dp_group* g, const int* members, const int* offsets, int n_sets) {
  return guarded([&]() -> int {
    if (g == nullptr || offsets == nullptr || n_sets < 1 || (members == nullptr && offsets[n_sets]))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_dp_group_prepare_sets: bad arguments");
    std::vector<std::vector<int>> sets;
    for (int i = 0; i < n_sets; ++i) {
      if (offsets[i + 1] < offsets[i])
        return set_error(EW_ERR_INVALID_ARGUMENT, "ew_dp_group_prepare_sets: offsets decrease");
      sets.emplace_back(members + offsets[i], members + offsets[i + 1]);
    }
    g->g->prepare(sets);
    return EW_OK;
  });
}

int ew_dp_group_recover(ew_dp_group* g, const int* departed, int n, int kind, void* old_buf,
                        void* replica, void* new_buf, int step, ew_stream_t stream,
                        ew_mttr_event* ev) {
  return guarded([&]() -> int {
    if (g == nullptr || n < 1 || departed == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_dp_group_recover: bad arguments");
    if (kind < 0 || kind > 3) return set_error(EW_ERR_INVALID_ARGUMENT, "bad event kind");
    elaskit::b200::RankBuffers b;
    b.old_buf = old_buf;
    b.replica = replica;
    b.new_buf = new_buf;
    const MttrEvent e = g->g->recover(std::vector<int>(departed, departed + n),
                                      static_cast<elaskit::EventKind>(kind), b, stream, step);
    to_c(e, ev);
    return EW_OK;
  });
}

int ew_dp_group_comm(const ew_dp_group* g, ew_comm** comm) {
  if (g == nullptr || comm == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  *comm = g->g->comm();
  return EW_OK;
}

int ew_dp_group_members(const ew_dp_group* g, int* out, int cap, int* n) {
  if (g == nullptr || n == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  const auto& m = g->g->members();
  *n = static_cast<int>(m.size());
  if (*n > cap) return set_error(EW_ERR_CAPACITY, "member buffer too small");
  std::copy(m.begin(), m.end(), out);
  return EW_OK;
}

int ew_dp_group_microbatches(const ew_dp_group* g, int* out, int cap, int* n) {
  if (g == nullptr || n == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  const auto& m = g->g->microbatch_sizes();
  *n = static_cast<int>(m.size());
  if (*n > cap) return set_error(EW_ERR_CAPACITY, "buffer too small");
  std::copy(m.begin(), m.end(), out);
  return EW_OK;
}

void ew_dp_group_free(ew_dp_group* g) { delete g; }

// -------------------------------------------------------- failure detector

int ew_detector_create(ew_channel* ch, const char* tag, double period_s, double timeout_s,
                       ew_detector** out) {
  return guarded([&]() -> int {
    if (ch == nullptr || tag == nullptr || out == nullptr)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_detector_create: bad arguments");
    elaskit::b200::DetectorOptions opt;
    opt.period_s = period_s;
    opt.timeout_s = timeout_s;
    *out = new ew_detector{std::make_unique<elaskit::b200::FailureDetector>(*ch->c, tag, opt)};
    return EW_OK;
  });
}

static int copy_members(const std::vector<int>& f, int* out, int cap, int* n) {
  *n = static_cast<int>(f.size());
  if (*n > cap) return set_error(EW_ERR_CAPACITY, "member buffer too small");
  std::copy(f.begin(), f.end(), out);
  return EW_OK;
}

int ew_detector_failed(const ew_detector* d, int* out, int cap, int* n) {
  if (d == nullptr || n == nullptr || (cap > 0 && out == nullptr))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_detector_failed: bad arguments");
  return copy_members(d->d->failed(), out, cap, n);
}

int ew_detector_wait(const ew_detector* d, double max_wait_s, int* out, int cap, int* n,
                     double* detect_s) {
  if (d == nullptr || n == nullptr || (cap > 0 && out == nullptr))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_detector_wait: bad arguments");
  return guarded([&]() -> int {
    double t = 0.0;
    const std::vector<int> f = d->d->wait_for_failure(max_wait_s, &t);
    if (detect_s) *detect_s = t;
    return copy_members(f, out, cap, n);
  });
}

int ew_detector_stop(ew_detector* d) {
  if (d == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL detector");
  d->d->stop_beating();
  return EW_OK;
}

void ew_detector_free(ew_detector* d) { delete d; }

// ------------------------------------------------------- in-place executor

int ew_inplace_exec_create(ew_channel* ch, const int64_t* layer_bytes, int n_layers,
                           const int* old_members, int n_old, const int* new_members, int n_new,
                           void* buf, void* replica, int64_t stage_bytes, int64_t phase_bytes,
                           int slack, int gather_streams, int flush_ctas, int64_t block_bytes,
                           double barrier_timeout_s, ew_inplace_exec** out) {
  return guarded([&]() -> int {
    if (ch == nullptr || layer_bytes == nullptr || n_layers < 1 || out == nullptr ||
        !old_members || !new_members || n_old < 1 || n_new < 1)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_inplace_exec_create: bad arguments");
    const ReshardPlan rp = ReshardPlan::build(
        std::vector<int64_t>(layer_bytes, layer_bytes + n_layers),
        std::vector<int>(old_members, old_members + n_old),
        std::vector<int>(new_members, new_members + n_new));
    elaskit::b200::InPlaceOptions opt;
    opt.stage_bytes = stage_bytes;
    opt.phase_bytes = phase_bytes;
    opt.slack = slack;
    opt.gather_streams = gather_streams;
    opt.flush_ctas = flush_ctas;
    opt.block_bytes = block_bytes;
    opt.barrier_timeout_s = barrier_timeout_s;
    *out = new ew_inplace_exec{std::make_unique<InPlaceExecutor>(*ch->c, rp, buf, replica, opt)};
    return EW_OK;
  });
}

int ew_inplace_exec_launch(ew_inplace_exec* x, uint64_t* block_sums, ew_stream_t stream) {
  return guarded([&]() -> int {
    if (x == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    x->x->launch(stream, block_sums);
    return EW_OK;
  });
}

int ew_inplace_exec_timed_out(const ew_inplace_exec* x, int* timed_out) {
  return guarded([&]() -> int {
    if (x == nullptr || timed_out == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    *timed_out = x->x->timed_out() ? 1 : 0;
    return EW_OK;
  });
}

int ew_inplace_exec_info(const ew_inplace_exec* x, int64_t* n_phases, int64_t* stage_alloc) {
  if (x == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  if (n_phases) *n_phases = static_cast<int64_t>(x->x->schedule().phases.size());
  if (stage_alloc) *stage_alloc = x->x->schedule().stage_alloc;
  return EW_OK;
}

void ew_inplace_exec_free(ew_inplace_exec* x) { delete x; }

// ------------------------------------------------------------ ring replicas

int ew_replay_replica_create(ew_channel* ch, const float* my_grad, const uint64_t* my_rows,
                             float* master, float* exp_avg, float* exp_avg_sq,
                             uint16_t* param_bf16, int64_t n, const void* image,
                             int64_t image_bytes, int64_t block_bytes, ew_replay_replica** out) {
  return guarded([&]() -> int {
    if (ch == nullptr || out == nullptr || !my_grad || !my_rows || !master || !exp_avg ||
        !exp_avg_sq || !param_bf16 || !image || n < 0 || image_bytes <= 0)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_replay_replica_create: bad arguments");
    elaskit::b200::AdamShard a;
    a.master = master;
    a.exp_avg = exp_avg;
    a.exp_avg_sq = exp_avg_sq;
    a.param_bf16 = param_bf16;
    a.n = n;
    a.image = image;
    a.image_bytes = image_bytes;
    *out = new ew_replay_replica{
        std::make_unique<elaskit::b200::ReplayReplica>(*ch->c, my_grad, my_rows, a, block_bytes)};
    return EW_OK;
  });
}

int ew_replay_replica_replay(ew_replay_replica* r, const ew_adam_hyper* hyper, int64_t step,
                             ew_stream_t stream) {
  return guarded([&]() -> int {
    if (r == nullptr || hyper == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    r->r->replay(*hyper, step, stream);
    return EW_OK;
  });
}

int ew_replay_replica_verify(const ew_replay_replica* r, uint32_t* bad_count, int reread,
                             ew_stream_t stream) {
  return guarded([&]() -> int {
    if (r == nullptr || bad_count == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    if (reread)
      r->r->verify_by_reread(bad_count, stream);
    else
      r->r->verify(bad_count, stream);
    return EW_OK;
  });
}

int ew_replay_replica_owner(const ew_replay_replica* r, int* owner) {
  if (r == nullptr || owner == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  *owner = r->r->owner();
  return EW_OK;
}

void ew_replay_replica_free(ew_replay_replica* r) { delete r; }

int ew_ring_replica_create(ew_channel* ch, const ew_layout* layout, const void* my_snap,
                           const uint64_t* my_rows, void* replica, int64_t block_bytes,
                           ew_ring_replica** out) {
  return guarded([&]() -> int {
    if (ch == nullptr || layout == nullptr || out == nullptr || !my_snap || !my_rows || !replica)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_ring_replica_create: bad arguments");
    *out = new ew_ring_replica{std::make_unique<elaskit::b200::RingReplica>(
        *ch->c, layout->layout, my_snap, my_rows, replica, block_bytes)};
    return EW_OK;
  });
}

int ew_ring_replica_refresh(const ew_ring_replica* r, uint32_t* bad_count, ew_stream_t stream) {
  return guarded([&]() -> int {
    if (r == nullptr || bad_count == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    r->r->refresh(bad_count, stream);
    return EW_OK;
  });
}

void ew_ring_replica_free(ew_ring_replica* r) { delete r; }

// ------------------------------------------------------- (d) over peers

int ew_peer_reduce_create(ew_channel* ch, const float* const* units, const double* weights,
                          int n_units, float* out, int64_t n, double barrier_timeout_s,
                          ew_peer_reduce** handle) {
  return guarded([&]() -> int {
    if (ch == nullptr || handle == nullptr || out == nullptr || n_units < 0 || n < 0 ||
        (n_units > 0 && (!units || !weights)))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_peer_reduce_create: bad arguments");
    *handle = new ew_peer_reduce{std::make_unique<elaskit::b200::PeerReduce>(
        *ch->c, std::vector<const float*>(units, units + n_units),
        std::vector<double>(weights, weights + n_units), out, n, barrier_timeout_s)};
    return EW_OK;
  });
}

int ew_peer_reduce_create_i64(ew_channel* ch, const int64_t* acc, float* out, int64_t n,
                              double barrier_timeout_s, ew_peer_reduce** handle) {
  return guarded([&]() -> int {
    if (ch == nullptr || handle == nullptr || out == nullptr || acc == nullptr || n < 0)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_peer_reduce_create_i64: bad arguments");
    *handle = new ew_peer_reduce{
        std::make_unique<elaskit::b200::PeerReduce>(*ch->c, acc, out, n, barrier_timeout_s)};
    return EW_OK;
  });
}

int ew_peer_reduce_scale(ew_peer_reduce* r, ew_stream_t stream, int* frac_bits) {
  return guarded([&]() -> int {
    if (r == nullptr || frac_bits == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    *frac_bits = r->r->scale(stream);
    return EW_OK;
  });
}

int ew_peer_reduce_run(ew_peer_reduce* r, int frac_bits, ew_stream_t stream) {
  return guarded([&]() -> int {
    if (r == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    r->r->run(frac_bits, stream);
    return EW_OK;
  });
}

int ew_peer_reduce_wait(ew_peer_reduce* r, ew_stream_t stream) {
  return guarded([&]() -> int {
    if (r == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    r->r->wait(stream);
    return EW_OK;
  });
}

int ew_peer_reduce_info(const ew_peer_reduce* r, int64_t* total_units, int* timed_out) {
  return guarded([&]() -> int {
    if (r == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    if (total_units) *total_units = r->r->total_units();
    if (timed_out) *timed_out = r->r->timed_out() ? 1 : 0;
    return EW_OK;
  });
}

void ew_peer_reduce_free(ew_peer_reduce* r) { delete r; }

// ------------------------------------------------------------ host images

int ew_host_images_create(ew_channel* ch, const ew_layout* layout, const char* tag,
                          const int* readable, int n_readable, int map_for_device,
                          ew_host_images** out) {
  return guarded([&]() -> int {
    if (ch == nullptr || layout == nullptr || tag == nullptr || out == nullptr ||
        n_readable < 0 || (n_readable > 0 && readable == nullptr))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_host_images_create: bad arguments");
    *out = new ew_host_images{std::make_unique<elaskit::b200::HostImages>(
        *ch->c, layout->layout, tag, std::vector<int>(readable, readable + n_readable),
        map_for_device != 0)};
    return EW_OK;
  });
}

int ew_host_images_publish(ew_host_images* h, const void* live, int64_t epoch, ew_stream_t stream,
                           int64_t* epoch_out) {
  return guarded([&]() -> int {
    if (h == nullptr || live == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    const int64_t e = h->h->publish(live, stream, epoch);
    if (epoch_out) *epoch_out = e;
    return EW_OK;
  });
}

int ew_host_images_commit_host(ew_host_images* h, int64_t epoch) {
  return guarded([&]() -> int {
    if (h == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    h->h->commit_host(epoch);
    return EW_OK;
  });
}

int ew_host_images_committed(const ew_host_images* h, int member, int64_t* epoch) {
  return guarded([&]() -> int {
    if (h == nullptr || epoch == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    *epoch = h->h->committed_epoch(member);
    return EW_OK;
  });
}

int ew_host_images_device_ptr(const ew_host_images* h, int member, void** ptr) {
  return guarded([&]() -> int {
    if (h == nullptr || ptr == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    *ptr = h->h->device_ptr(member);
    return EW_OK;
  });
}

int ew_host_images_host_ptr(const ew_host_images* h, int member, int64_t epoch, void** ptr,
                            int64_t* bytes) {
  return guarded([&]() -> int {
    if (h == nullptr || ptr == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    *ptr = h->h->host_ptr(member, epoch);
    if (bytes) *bytes = h->h->image_bytes(member);
    return EW_OK;
  });
}

void ew_host_images_free(ew_host_images* h) { delete h; }

// ------------------------------------------------------- layer migration

int ew_layer_migration_create(ew_channel* ch, int source, int target, void* params,
                              int64_t param_bytes, int64_t* acc, int64_t n, int transfer_ctas,
                              double barrier_timeout_s, ew_layer_migration** out) {
  return guarded([&]() -> int {
    if (ch == nullptr || out == nullptr || params == nullptr || acc == nullptr || n < 0 ||
        param_bytes < 0)
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_layer_migration_create: bad arguments");
    *out = new ew_layer_migration{std::make_unique<elaskit::b200::LayerMigration>(
        *ch->c, source, target, params, param_bytes, acc, n, transfer_ctas, barrier_timeout_s)};
    return EW_OK;
  });
}

int ew_layer_migration_step(ew_layer_migration* m, int what, ew_stream_t stream) {
  return guarded([&]() -> int {
    if (m == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    switch (what) {
      case 0: m->m->pull_params(stream); break;
      case 1: m->m->shadow_done(stream); break;
      case 2: m->m->prefetch_payback(stream); break;
      case 3: m->m->payback(stream); break;
      default: return set_error(EW_ERR_INVALID_ARGUMENT, "unknown migration step");
    }
    return EW_OK;
  });
}

int ew_layer_migration_run(ew_layer_migration* m, int target_side, const float* const* units,
                           const double* weights, int n_units, int64_t n, int frac_bits, int k,
                           ew_stream_t compute, ew_stream_t transfer) {
  return guarded([&]() -> int {
    if (m == nullptr || n_units < 0 || (n_units > 0 && (!units || !weights)))
      return set_error(EW_ERR_INVALID_ARGUMENT, "ew_layer_migration_run: bad arguments");
    const std::vector<const float*> u(units, units + n_units);
    const std::vector<double> w(weights, weights + n_units);
    if (target_side)
      m->m->run_target(u, w, n, frac_bits, k, compute, transfer);
    else
      m->m->run_shadow(u, w, n, frac_bits, k, compute);
    return EW_OK;
  });
}

int ew_layer_migration_info(const ew_layer_migration* m, const int64_t** payback_buffer,
                            int* timed_out) {
  return guarded([&]() -> int {
    if (m == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
    if (payback_buffer) *payback_buffer = m->m->payback_buffer();
    if (timed_out) *timed_out = m->m->timed_out() ? 1 : 0;
    return EW_OK;
  });
}

void ew_layer_migration_free(ew_layer_migration* m) { delete m; }

}  // extern "C"
