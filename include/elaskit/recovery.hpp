// Multi-process DP recovery on B200 — the executed counterpart of the
// reference's Simulation::recover_elaswave DP slice (sim.cpp:597-722), which
// only prices the steps (comm_edit_time sim.cpp:436-450, remap_time
// sim.cpp:452-483) and fills MttrEvent (sim.hpp:31-45) / mttr.csv
// (sim.cpp:1119-1132).
//
// One process per GPU (or, for tests, several processes sharing one GPU:
// CUDA IPC maps a peer process's allocation on the same device too).  The
// ranks of a DP group meet through a pluggable key-value Store (a TCP store
// ships in the library; a caller can plug its own, e.g. torch.distributed's
// c10d store through the C ABI).  The store carries plumbing only — CUDA IPC
// handles, barriers, per-rank verdict counts; every byte of model state and
// every checksum moves GPU to GPU through peer pointers.
//
//   Store / Channel      rendezvous: set/get + allgather/barrier over members
//   PeerBuffers          every member's OLD / REPLICA / NEW / block-sum arrays,
//                        IPC-mapped once (steady state) for the copy kernels
//   ReshardExecutor      plan (interleaved_layout + integrity_check +
//                        overlap_matrix) -> this GPU's pull program ->
//                        one launch that checksums what it lands
//   BlockVerifier        global checksum conservation: sum over survivors of
//                        landed block sums == sum of the source's block sums,
//                        reduce-scattered over peer memory, verdicts via Store
//   PreparedRecovery     every single departure planned, lowered and bound in
//                        steady state: recover(d) = comm lookup + one launch
//                        + one verification
//   DpGroup              the membership owner: plan_edit, the prepared NCCL
//                        communicators (comm repair = lookup), reshaper,
//                        recovery, MttrEvent
//   InPlaceExecutor      staged in-place reshard (config D): OLD and NEW in
//                        one buffer, phases behind device-side barriers
#pragma once

#include <atomic>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "elaskit/b200.hpp"
#include "elaskit/cluster.hpp"
#include "elaskit/communicator.hpp"
#include "elaskit/migration.hpp"
#include "elaskit/param_fabric.hpp"
#include "ew_api.h"

namespace elaskit::b200 {

// ---------------------------------------------------------------- rendezvous

// Blocking key-value store shared by the ranks (the out-of-band channel).
// get() waits until the key is set; implementations throw
// std::runtime_error on timeout.
class Store {
 public:
  virtual ~Store() = default;
  virtual void set(const std::string& key, const std::string& value) = 0;
  virtual std::string get(const std::string& key) = 0;
  // drop a key nobody will read again (default: keep it)
  virtual void erase(const std::string& key) { (void)key; }
};

// TCP store: rank `is_server` hosts it on host:port (a listening thread), every
// process (the host included) talks to it over one connection.
std::unique_ptr<Store> tcp_store(const std::string& host, int port, bool is_server,
                                 double timeout_s = 300.0);

// Store over caller callbacks (the C ABI's ew_store_callbacks); `erase` may
// be empty.
std::unique_ptr<Store> callback_store(std::function<void(const std::string&, const std::string&)> set,
                                      std::function<std::string(const std::string&)> get,
                                      std::function<void(const std::string&)> erase = {});

// Collective operations among an ordered member list over a Store.  Every
// member issues the same sequence of calls; a per-channel counter names the
// keys, so channels with distinct `name`s never collide.  A member erases
// its key of round k-1 once it has completed round k (every member has then
// set its round-k key, so nobody still reads round k-1): the store holds at
// most two rounds per channel.
class Channel {
 public:
  Channel(Store& store, std::string name, std::vector<int> members, int me);
  const std::vector<int>& members() const { return members_; }
  int me() const { return me_; }
  int index() const { return index_; }
  const std::string& name() const { return name_; }
  // every member's blob, in member order
  std::vector<std::string> allgather(const std::string& mine);
  void barrier() { allgather(std::string()); }
  std::int64_t sum(std::int64_t mine);
  Store& store() { return store_; }

 private:
  Store& store_;
  std::string name_;
  std::vector<int> members_;
  int me_ = -1, index_ = -1;
  std::uint64_t seq_ = 0;
};

// ------------------------------------------------------------ peer buffers

// Buffers one rank contributes to a reshard (device pointers, caller-owned;
// null where the rank has none).  Roles as BufRole (Old/Replica/New).
struct RankBuffers {
  void* old_buf = nullptr;
  void* replica = nullptr;
  void* new_buf = nullptr;
};

// Device buffers of every member keyed by (role, member), IPC-mapped in this
// process (own buffers entered as is).  Exchange once, look up many times.
class PeerBuffers {
 public:
  PeerBuffers() = default;
  ~PeerBuffers();
  PeerBuffers(const PeerBuffers&) = delete;
  PeerBuffers& operator=(const PeerBuffers&) = delete;

  // Collective over `ch`: publish `mine` (key -> local device pointer) and
  // map every other member's entries whose key passes `want` (all if empty).
  void exchange(Channel& ch, const std::map<int, void*>& mine,
                const std::function<bool(int key, int member)>& want = {});
  void* get(int key, int member) const;  // nullptr if absent
  bool has(int key, int member) const { return get(key, member) != nullptr; }
  void put(int key, int member, void* p) { table_[{key, member}] = p; }
  void close();

 private:
  std::map<std::pair<int, int>, void*> table_;
  std::vector<void*> opened_;
};

// ---------------------------------------------------------------- reshard

// One membership change of an interleaved-ZeRO DP group, planned exactly as
// the reference plans it: integrity_check + overlap_matrix on the interleaved
// layouts (A4, A6, A7), the departed ranks' bytes sourced from their ring
// holders (SnapshotRing over the old members).
struct ReshardPlan {
  std::vector<std::int64_t> layer_bytes;
  std::vector<int> old_members, new_members;
  std::set<int> failed;
  PartitionLayout src, dst;
  SnapshotRing ring;
  TransferPlan plan;
  double plan_seconds = 0.0;

  static ReshardPlan build(const std::vector<std::int64_t>& layer_bytes,
                           std::vector<int> old_members, std::vector<int> new_members);
  // Arbitrary layouts (e.g. a cross-stage layer move); ring_members empty:
  // no ring (no failed members allowed).  integrity_check when failed.
  static ReshardPlan from_layouts(PartitionLayout src, PartitionLayout dst, std::set<int> failed,
                                  std::vector<int> ring_members);
  // member whose OLD shard `holder` keeps (-1 if none)
  int replica_of(int holder) const;
  std::int64_t n_blocks(std::int64_t block_bytes) const {
    return (src.total_bytes + block_bytes - 1) / block_bytes;
  }
};

// This GPU's share of a reshard: pull copies landing in its NEW buffer,
// verified on arrival (the landed bytes' block sums are added to a device
// array), or push copies sourced from its buffers.  Peer pointers come from
// a PeerBuffers table.
class ReshardExecutor {
 public:
  // local_replica (pull): copies the plan sources from the OLD shard of the
  // member this rank backs up read this rank's own replica of it instead
  // (b200::prefer_local_replica); the peer table must then hold this rank's
  // REPLICA buffer, kept current by the ring replica.
  ReshardExecutor(const ReshardPlan& rp, int me, bool push = false,
                  std::int64_t block_bytes = 65536, bool local_replica = false);
  ~ReshardExecutor();
  ReshardExecutor(const ReshardExecutor&) = delete;
  ReshardExecutor& operator=(const ReshardExecutor&) = delete;

  // Build the program; every (role, member) a copy touches must be in
  // `peers` (own buffers included).  verify (pull only): checksum what
  // lands.  Throws std::runtime_error naming a missing peer buffer.
  void bind(const PeerBuffers& peers, bool verify);
  // block_sums: device u64 [2 * n_blocks] (caller-zeroed) when verified;
  // abort_flag: optional device int vetoing the launch (peer barrier error)
  void launch(ew_stream_t stream, std::uint64_t* block_sums = nullptr,
              const int* abort_flag = nullptr, int n_ctas = 0, int remote_ctas = 0) const;
  // (role, member) pairs the program reads or writes on other GPUs
  std::set<std::pair<int, int>> peers_needed() const;
  std::int64_t new_bytes() const;
  bool bound() const { return prog_ != nullptr; }
  const ReshardPlan& plan() const { return rp_; }

 private:
  ReshardPlan rp_;
  int me_;
  bool push_;
  std::int64_t block_bytes_;
  std::vector<CopyDesc> copies_;
  ew_shardmap* new_map_ = nullptr;
  ew_copy_program* prog_ = nullptr;
};

// Global checksum conservation over peer memory.  Every survivor holds three
// device arrays of 2 * n_blocks u64: `landed` (its verified copy's block
// sums), `old_blocks` (the block sums of its own OLD shard, from the per-step
// snapshot rows) and `replica_blocks` (its ring replica's).  Conservation:
//   sum_r landed_r == sum_r old_blocks_r + replica_blocks_{holder of d}
// checked on slice [lo, hi) of the blocks by each survivor (a reduce-scatter
// over NVLink reads), mismatch counts summed over the Store.
class BlockVerifier {
 public:
  BlockVerifier() = default;
  ~BlockVerifier();
  BlockVerifier(const BlockVerifier&) = delete;
  BlockVerifier& operator=(const BlockVerifier&) = delete;
  // plus / minus: device arrays (local or peer) to add / subtract
  void set(const std::vector<const std::uint64_t*>& plus,
           const std::vector<const std::uint64_t*>& minus, std::int64_t n_words,
           std::int64_t lo, std::int64_t hi);
  // enqueue the slice check; *bad_dev (device u32) receives the mismatches
  void run(ew_stream_t stream, std::uint32_t* bad_dev) const;

 private:
  ew_block_verifier* v_ = nullptr;
};

// ------------------------------------------------------------ ring replicas

// The AdamW state of one ZeRO shard as the replay kernel updates it: device
// pointers into one byte image (the Python device.AdamState layout: fp32
// master, exp_avg, exp_avg_sq and the bf16 parameter copy, sections on
// 1 MiB boundaries).
struct AdamShard {
  float* master = nullptr;
  float* exp_avg = nullptr;
  float* exp_avg_sq = nullptr;
  std::uint16_t* param_bf16 = nullptr;
  std::int64_t n = 0;
  const void* image = nullptr;
  std::int64_t image_bytes = 0;
};

// Ring replica kept by optimizer replay (the paper's
// mechanism, with the replica in the holder's HBM): each
// step the holder applies the owner's AdamW step to its replica, reading the
// owner's reduced gradient shard over NVLink (4 B/param instead of the
// 14 B/param of a state pull), and produces the replica's checksum rows in the
// same pass; verification compares them with the owner's rows in the owner's
// HBM.  Both sides run the same explicitly rounded kernel on the same inputs,
// so the replica stays byte-identical.  Ordering contract: the owner must not
// overwrite its gradient shard before the holder's replay of that step
// finished.
class ReplayReplica {
 public:
  // Collective over `ch` (the ring's members in ring order = ascending ids).
  // my_grad / my_rows: this rank's gradient shard and the checksum rows of
  // its own state (written by its ew_adam_step_rows); replica: the state of
  // the member this rank backs up (SnapshotRing::backs_up).
  ReplayReplica(Channel& ch, const float* my_grad, const std::uint64_t* my_rows,
                AdamShard replica, std::int64_t block_bytes = 65536);
  ~ReplayReplica();
  ReplayReplica(const ReplayReplica&) = delete;
  ReplayReplica& operator=(const ReplayReplica&) = delete;

  int owner() const { return owner_; }
  // the owner's step `step` applied to the replica (+ its rows, one pass)
  void replay(const ew_adam_hyper& hyper, std::int64_t step, ew_stream_t stream);
  // *bad_dev = rows where the replica's rows differ from the owner's
  void verify(std::uint32_t* bad_dev, ew_stream_t stream) const;
  // stronger: recompute the replica's rows from HBM and compare
  void verify_by_reread(std::uint32_t* bad_dev, ew_stream_t stream) const;
  const std::uint64_t* replica_rows() const { return rows_; }

 private:
  PeerBuffers peers_;
  AdamShard rep_;
  int owner_ = -1;
  std::int64_t block_bytes_;
  std::int64_t n_rows_ = 0;
  std::uint64_t* rows_ = nullptr;
  const float* owner_grad_ = nullptr;
  const std::uint64_t* owner_rows_ = nullptr;
  ew_shardmap* map_ = nullptr;
};

// Ring replica by a full pull of the owner's per-step snapshot (for
// optimizers the library does not own): the staged copy over NVLink, then
// kernel (a)'s verification of the replica against the owner's rows, read
// in the owner's HBM.
class RingReplica {
 public:
  // Collective over `ch`.  layout: the source layout (the packing of every
  // member's shard); my_snap / my_rows: this rank's snapshot and its rows;
  // replica: buffer for the owner's shard.
  RingReplica(Channel& ch, const PartitionLayout& layout, const void* my_snap,
              const std::uint64_t* my_rows, void* replica, std::int64_t block_bytes = 65536);
  ~RingReplica();
  RingReplica(const RingReplica&) = delete;
  RingReplica& operator=(const RingReplica&) = delete;

  int owner() const { return owner_; }
  // pull the owner's snapshot into the replica and verify it (*bad_dev)
  void refresh(std::uint32_t* bad_dev, ew_stream_t stream) const;

 private:
  PeerBuffers peers_;
  int owner_ = -1;
  void* replica_ = nullptr;
  const std::uint64_t* owner_rows_ = nullptr;
  ew_shardmap* map_ = nullptr;
  ew_copy_program* copy_ = nullptr;
};

// ------------------------------------------------------- layer migration

// Non-blocking layer migration with shadow-gradient payback (
// the reference plans it, plan_layer_migration migration.cpp:9-61, and only
// models its time, Simulation::migrate sim.cpp:485-530).  The target pulls
// the layer's parameters over NVLink with a few CTAs on a low-priority
// stream; the source's shadow instance folds micro-batches [0, k) into its
// int64 accumulator and releases a device barrier; the target then pulls
// that accumulator and adds it inside its last fold (ew_weighted_fold_addend).
// Integer sums: the migrated step's gradient is bit-identical to the static
// step's for every k.
class LayerMigration {
 public:
  // Collective over `ch` = {source, target}.  Source: `params` is its layer's
  // parameter buffer, `acc` its shadow accumulator.  Target: `params` is the
  // destination buffer, `acc` its own accumulator (n int64 each).
  LayerMigration(Channel& ch, int source, int target, void* params, std::int64_t param_bytes,
                 std::int64_t* acc, std::int64_t n, int transfer_ctas = 32,
                 double barrier_timeout_s = 30.0);
  ~LayerMigration();
  LayerMigration(const LayerMigration&) = delete;
  LayerMigration& operator=(const LayerMigration&) = delete;

  // target: the parameter pull on `stream` (low priority by convention)
  void pull_params(ew_stream_t stream);
  // source: after the shadow instance's last fold
  void shadow_done(ew_stream_t stream);
  // target: wait (on `stream`) for the source's shadow_done, then pull its
  // accumulator into payback_buffer()
  void prefetch_payback(ew_stream_t stream);
  // target, unoverlapped: acc += the source's accumulator, read in peer HBM
  void payback(ew_stream_t stream);
  // The target's step for the layer: micro-batches [0, k) without it, the
  // parameter wait before k, folds [k, M) into acc, the payback in the last
  // fold.  `compute` / `transfer`: cudaStream_t.
  void run_target(const std::vector<const float*>& units, const std::vector<double>& weights,
                  std::int64_t n, int frac_bits, int k, ew_stream_t compute, ew_stream_t transfer);
  // The source's shadow instance: folds [0, k) into acc, then shadow_done.
  void run_shadow(const std::vector<const float*>& units, const std::vector<double>& weights,
                  std::int64_t n, int frac_bits, int k, ew_stream_t compute);
  const std::int64_t* payback_buffer() const { return payback_; }
  bool timed_out() const;

 private:
  int me_, source_, target_, transfer_ctas_;
  double timeout_s_;
  std::int64_t* acc_;
  std::int64_t n_;
  PeerBuffers peers_;
  ew_copy_program* pull_ = nullptr;
  ew_copy_program* payback_pull_ = nullptr;
  std::int64_t* payback_ = nullptr;
  const std::int64_t* source_acc_ = nullptr;
  ew_peer_barrier* barrier_ = nullptr;
  unsigned long long* flags_ = nullptr;
};

// ------------------------------------------------------------ host images

// Host-memory images of every member's shard — the reference's
// Medium::H2D_D2D source (param_fabric.hpp:59-79; the paper keeps the
// replica in host DRAM).  One POSIX shm segment per member
// ("/ew_<tag>_<member>": a header page with the committed epoch, then two
// image slots), pinned and mapped for this GPU (ew_host_register).  The owner
// publishes its shard each step with a D2H into the slot of epoch e (e mod
// 2) followed, in stream order, by the commit word; a publish torn by a crash
// leaves the previous epoch's image in use.  At recovery the holder's REPLICA
// entry of the copy table points at the departed member's committed image,
// so the destinations' copy kernels read those bytes from host memory over
// their own PCIe links.  An image outlives its owner process.
class HostImages {
 public:
  static constexpr std::int64_t kPage = 4096;
  // Collective over `ch`.  readable: members whose images this rank maps
  // (default all; its own always).  map_for_device = false skips the pinning
  // (host-side users, CPU tests): device_ptr() then returns host addresses.
  HostImages(Channel& ch, const PartitionLayout& layout, const std::string& tag,
             const std::vector<int>& readable = {}, bool map_for_device = true);
  ~HostImages();
  HostImages(const HostImages&) = delete;
  HostImages& operator=(const HostImages&) = delete;

  // D2H of this member's live shard into the slot of `epoch` (default: the
  // next one), then the commit word, both on `stream`.  Returns the epoch.
  std::int64_t publish(const void* live, ew_stream_t stream, std::int64_t epoch = -1);
  // host-side commit (a publisher without a GPU copy, tests)
  void commit_host(std::int64_t epoch);
  std::int64_t committed_epoch(int member) const;  // -1: none yet
  // device address of member's last committed image (throws if none)
  void* device_ptr(int member) const;
  // host address of member's image of `epoch` (default: committed)
  std::uint8_t* host_ptr(int member, std::int64_t epoch = -1) const;
  std::int64_t image_bytes(int member) const { return bytes_.at(member); }
  std::int64_t slot_bytes(int member) const { return slot_.at(member); }

 private:
  struct Segment {
    std::uint8_t* addr = nullptr;
    std::int64_t size = 0;
    std::uint8_t* dev = nullptr;
    std::vector<void*> pieces;  // registrations (unregistered at close)
  };
  void map_member(int member, bool create);
  void release();
  int me_;
  std::string tag_;
  bool map_for_device_;
  std::map<int, std::int64_t> bytes_, slot_;
  std::map<int, Segment> segs_;
  std::int64_t next_epoch_ = -1;
};

// ------------------------------------------------------ failure detection

// Heartbeat failure detector for the processes of one node's DP group (the
// reference's detection is the constant detect_s, presets.hpp:63, used at
// sim.cpp:601; the paper omits its agent).  Each member's beat thread proves
// its device still executes work — a 4-byte H2D copy on a private stream
// (a copy engine: the job's long kernels do not delay it), then a stream
// synchronise — and only then publishes (beat count, CLOCK_MONOTONIC time)
// in its slot of a node-shared POSIX shm segment; a member whose slot stops
// advancing for timeout_s is failed (a dead process, or a live one whose
// device no longer completes work).  Watching reads host memory only: no
// CUDA call touches a failed peer.  detect_s of a verdict = time from the
// failed member's last heartbeat to the verdict (an upper bound on the time
// since it failed).
struct DetectorOptions {
  double period_s = 0.001;   // beat interval
  double timeout_s = 0.02;   // silence that fails a member
};

class FailureDetector {
 public:
  // Collective over `ch` (segment creation and attach); starts beating.
  FailureDetector(Channel& ch, const std::string& tag, DetectorOptions opt = {});
  ~FailureDetector();
  FailureDetector(const FailureDetector&) = delete;
  FailureDetector& operator=(const FailureDetector&) = delete;

  // Members silent for more than timeout_s now (ascending), with the age of
  // each one's last heartbeat.
  std::vector<int> failed(std::vector<double>* silence_s = nullptr) const;
  // Block until at least one member fails or max_wait_s passes; returns the
  // failed members and *detect_s (seconds from the first failed member's
  // last heartbeat to this verdict).
  std::vector<int> wait_for_failure(double max_wait_s, double* detect_s) const;
  // Stop this member's beats (fault injection: a silent member).
  void stop_beating();

 private:
  void beat_loop();
  std::vector<int> members_;
  int me_;
  std::string name_;
  DetectorOptions opt_;
  void* shm_ = nullptr;
  std::size_t shm_bytes_ = 0;
  bool owner_ = false;
  std::atomic<bool> stop_{false};
  std::thread beater_;
};

// ------------------------------------------------- (d) over peer memory

// The gradient-scale-preserving weighted reduce fused with
// its collective over peer memory — no NCCL: each rank quantises its slice
// of every rank's contribution units (read from peer HBM, TMA-staged) and
// sums int64 (reduce-scatter), then pulls the other slices (all-gather),
// between stream-ordered device barriers.  The fixed-point scale comes from
// the global absmax (a local kernel, then one double per rank over the
// channel).  Bit-identical to the NCCL int64 path and to one GPU folding
// every unit, for any world size and split.  Reference: weighted_grad_average
// (dataflow.cpp:71-83), the toy fold (sim.cpp:901-953).
class PeerReduce {
 public:
  // fp32 units: this rank's units (n elements each) and weights, and its fp32
  // output.  Collective over `ch`.
  PeerReduce(Channel& ch, const std::vector<const float*>& units,
             const std::vector<double>& weights, float* out, std::int64_t n,
             double barrier_timeout_s = 30.0);
  // int64 accumulators: each rank folded its own units into `acc`
  // (ew_weighted_fold, accumulate=1); the collective sums accumulators.
  PeerReduce(Channel& ch, const std::int64_t* acc, float* out, std::int64_t n,
             double barrier_timeout_s = 30.0);
  ~PeerReduce();
  PeerReduce(const PeerReduce&) = delete;
  PeerReduce& operator=(const PeerReduce&) = delete;

  std::int64_t total_units() const { return total_units_; }
  // fixed-point bits of the global unit set (fp32-unit form): the local
  // weighted absmax, the max over ranks, ew_fixed_point_bits.  Synchronises
  // `stream` once.
  int scale(ew_stream_t stream);
  // barrier -> reduce-scatter -> barrier -> all-gather, all stream-ordered
  void run(int frac_bits, ew_stream_t stream);
  // trailing barrier: nobody frees buffers a peer may still read
  void wait(ew_stream_t stream);
  bool timed_out() const;

 private:
  void connect(Channel& ch, std::map<int, void*> mine, const std::string& extra);
  Channel& ch_;
  std::int64_t n_ = 0;
  std::int64_t total_units_ = 0;
  std::vector<const float*> units_;
  std::vector<double> weights_;
  PeerBuffers peers_;
  ew_peer_fold* fold_ = nullptr;
  ew_peer_barrier* barrier_ = nullptr;
  unsigned long long* flags_ = nullptr;
  double* dmax_ = nullptr;
  double timeout_s_;
};

// ------------------------------------------------------------ MTTR record

// Reference MttrEvent (sim.hpp:31-45) with measured seconds.
struct MttrEvent {
  int step = 0;
  double t_event_s = 0.0;
  std::string kind = "fail_stop";
  double detect_s = 0.0;          // detection: the agent's, outside this library
  double comm_repair_s = 0.0;     // plan_edit + NCCL communicator repair
  double remap_s = 0.0;           // copy + verification
  double migration_stall_s = 0.0; // no layer migration on the DP path
  double other_s = 0.0;           // micro-batch reshape + bookkeeping
  double lost_work_s = 0.0;
  bool verified = false;
  std::map<std::string, double> phases;
  double total_s() const {
    return detect_s + comm_repair_s + remap_s + migration_stall_s + other_s;
  }
};
// mttr.csv of the reference (sim.cpp:1119-1132)
std::string mttr_csv_header();
std::string mttr_csv_row(int index, const MttrEvent& ev);

// ------------------------------------------------------- prepared recovery

// Every single departure of a DP group planned, lowered and bound before it
// happens (steady state): the layouts, every peer's live shard and the ring
// replicas are known, so each rank builds, once, the verified pull program
// for each possible departed member d against one NEW buffer sized for the
// largest case, and maps every peer's verification arrays.  recover(d) is a
// table lookup, one copy launch and one verification.
struct PreparedOptions {
  std::int64_t block_bytes = 65536;
  double barrier_timeout_s = 30.0;
  // replica-aware sourcing (ReshardExecutor local_replica): valid while the
  // replicas are current (the per-step replay keeps them byte-identical; a
  // stale replica is caught by the conservation check)
  bool local_replicas = false;
};

class PreparedRecovery {
 public:
  // old_buf: this rank's live shard (source layout); replica: the shard of
  // the member it backs up (SnapshotRing::backs_up); old_rows / replica_rows:
  // their checksum rows (per-step snapshot rows; nullptr = computed here).
  // new_buf: caller-owned NEW buffer of new_capacity bytes (nullptr: the
  // object allocates one sized for the largest departure).  Collective over
  // `ch` (all members).
  PreparedRecovery(Channel& ch, const std::vector<std::int64_t>& layer_bytes, void* old_buf,
                   const std::uint64_t* old_rows, void* replica,
                   const std::uint64_t* replica_rows, void* new_buf = nullptr,
                   std::int64_t new_capacity = 0, PreparedOptions opt = {});
  ~PreparedRecovery();
  PreparedRecovery(const PreparedRecovery&) = delete;
  PreparedRecovery& operator=(const PreparedRecovery&) = delete;

  // Survivors only, all of them: copy the departed member's share into NEW,
  // verify by conservation.  Returns the verdict; phases (seconds) in `ev`.
  // stale_snapshot: this rank's state is not of the event's step (counted
  // into the verdict, which then fails)
  bool recover(int departed, ew_stream_t stream, MttrEvent* ev = nullptr,
               bool stale_snapshot = false);
  void* new_buf() const { return new_buf_; }
  std::int64_t new_bytes(int departed) const;
  const ReshardPlan& plan(int departed) const { return *plans_.at(departed); }
  const std::vector<int>& members() const { return members_; }

 private:
  Channel& ch_;
  std::vector<int> members_;
  int me_;
  PreparedOptions opt_;
  std::int64_t n_words_ = 0;
  void* new_buf_ = nullptr;
  bool own_new_ = true;
  std::uint64_t *landed_ = nullptr, *old_blocks_ = nullptr, *replica_blocks_ = nullptr;
  std::uint32_t* bad_ = nullptr;
  std::map<int, std::unique_ptr<ReshardPlan>> plans_;
  std::map<int, std::unique_ptr<ReshardExecutor>> execs_;
  std::map<int, std::unique_ptr<BlockVerifier>> verifiers_;
  std::map<int, std::unique_ptr<Channel>> survivors_;   // departed -> survivor channel
  std::map<int, ew_peer_barrier*> barriers_;            // departed -> survivor barrier
  PeerBuffers peers_;
  unsigned long long* flags_ = nullptr;  // u64 [n][n]: region d for departure d

  void release();
};

// The DP group as one rank sees it: members, communication links, the NCCL
// communicator of the (d) reduce, and micro-batch assignment.  recover()
// runs the reference's order (comm repair, dataflow, remap) and returns the
// measured MttrEvent.
struct DpGroupOptions {
  int per_slot_mbs = 4;
  int num_microbatches = 32;
  std::int64_t block_bytes = 65536;
  bool prepare_comms = true;  // one shrunk communicator per possible departure
  // ncclCommSplit splitShare for the prepared communicators: less memory,
  // but NCCL then requires the sibling communicators never to run
  // concurrently (prepare() serialises their warm-up either way)
  bool share_comm_resources = false;
};

class DpGroup {
 public:
  // comm: the group's NCCL communicator over `members` in ascending order
  // (nullptr: no (d) collective, e.g. processes sharing one GPU).  Takes
  // ownership.  Collective over ch when prepare_comms (ncclCommSplit per
  // departure, done in steady state).
  DpGroup(Channel& ch, const std::vector<std::int64_t>& layer_bytes, ew_comm* comm,
          DpGroupOptions opt = {});
  // A process outside the group that joins it at a ScaleOut (a device from
  // the free pool, cluster.hpp): it meets the members on `store` under the
  // members' group channel name `group_name`, with the group's current
  // `members`.  It has no communicator, shard or micro-batches until
  // recover(joiners, EventKind::ScaleOut, ...), where it learns them.
  DpGroup(Store& store, std::string group_name, const std::vector<std::int64_t>& layer_bytes,
          std::vector<int> members, int me, DpGroupOptions opt = {});
  ~DpGroup();
  DpGroup(const DpGroup&) = delete;
  DpGroup& operator=(const DpGroup&) = delete;

  // Attach a prepared recovery (steady state; borrowed) — single departures
  // then run its programs instead of planning at failure time.
  void attach(PreparedRecovery* prepared) { prepared_ = prepared; }
  // Survivors call this for a FailStop / ScaleIn of `departed`.  bufs: this
  // rank's OLD / REPLICA / NEW buffers for the change when not prepared.
  // ScaleOut (the reference's rejoin, sim.cpp:608,676-677): `departed` names
  // the joiners, and every member and every joiner calls it — members pass
  // OLD (their shard) and NEW, joiners NEW only.  Comm repair adds the
  // joiners' links (plan_edit) and builds the grown NCCL communicator (a
  // standby one from prepare_join when every participant has it, else
  // ncclCommInitRank now); the micro-batches are re-dealt over the grown
  // group; the members' shards are re-cut over it by one verified pull
  // program per GPU.  `step` names the event: the same (step, membership
  // change) must not recur within one group.
  MttrEvent recover(const std::vector<int>& departed, EventKind kind, const RankBuffers& bufs,
                    ew_stream_t stream, int step = 0);
  // Steady state before an expected ScaleOut (standby devices): build and
  // warm the grown communicator over members ∪ joiners now, so the join's
  // comm repair is a lookup; when the members premapped, the joiners map
  // the members' buffers now too.  Collective over members and joiners;
  // calls pair up in order per grown membership (the n-th call of a member
  // meets the n-th call of the joiners' group objects for that membership).
  void prepare_join(const std::vector<int>& joiners);
  // Steady state: map every member's OLD shard and replica (what a pull
  // program reads) and the verification arrays once, so an event planned at
  // failure time (a departure set without a PreparedRecovery, a ScaleOut)
  // pays no CUDA IPC mapping on its critical path.  Used by an event whose
  // participants all pass the buffers they premapped (agreed over the
  // store); otherwise the event maps as before.  old_rows / replica_rows:
  // the per-step snapshot's checksum rows of those buffers (device arrays
  // the caller refreshes in place every step); the event then takes its
  // source block sums from them instead of re-reading the shards.  The
  // buffers must stay allocated until the next premap or the group's end
  // (peers hold IPC mappings of them; a buffer freed and reallocated at the
  // same address would be read stale — verification on arrival then fails
  // the event rather than passing wrong bytes).  Collective over the members.
  void premap(const RankBuffers& bufs, const std::uint64_t* old_rows = nullptr,
              const std::uint64_t* replica_rows = nullptr);
  // Steady state, local: lower and bind this rank's verified pull program
  // for one expected event (a departure set, kind FailStop/ScaleIn, or the
  // joiners of a ScaleOut) into `new_buf`, over the premapped buffers.  The
  // event then only launches it.  After premap (members) / prepare_join
  // (joiners); a departing member has nothing to prepare.
  void prepare_move(EventKind kind, const std::vector<int>& targets, void* new_buf);
  // (Re)build one shrunk communicator per possible single departure of the
  // current membership (ncclCommSplit, splitShare) and run one collective on
  // each: steady-state work, collective over the members.  The constructor
  // calls it when opt.prepare_comms.  A departure whose set was prepared
  // repairs by lookup; any other by ncclCommShrink at failure time.
  void prepare();
  // The same for the given departure sets (e.g. config C's two non-adjacent
  // members leaving together): one shrunk communicator per set.
  void prepare(const std::vector<std::vector<int>>& departures);
  // The step whose state this member's OLD shard and replica hold — the
  // snapshot ring's step_tag (param_fabric.hpp:42), documented to equal the
  // current step but never checked by the reference.  Once set
  // (>= 0), an event at another `step` counts this member as stale in the
  // verdict: MttrEvent.verified is false, phases["stale_snapshots"] > 0.
  void set_snapshot_step(std::int64_t step) { snapshot_step_ = step; }
  ew_comm* comm() const { return comm_; }
  const std::vector<int>& members() const { return members_; }
  const std::vector<int>& microbatch_sizes() const { return mb_sizes_; }

 private:
  MttrEvent admit(const std::vector<int>& joiners, const RankBuffers& bufs, ew_stream_t stream,
                  int step);
  void commit_members(std::vector<int> next);
  struct Premap;
  std::unique_ptr<Premap> pm_;

  Store& store_;
  std::string name_;
  int me_;
  Channel* ch_;                      // over members_: the caller's, after a change owned
  std::unique_ptr<Channel> own_ch_;
  std::vector<std::int64_t> layer_bytes_;
  std::vector<int> members_;
  std::vector<int> mb_sizes_;
  std::set<Link> links_;
  ew_comm* comm_ = nullptr;
  std::map<std::vector<int>, ew_comm*> prepared_comms_;  // departed set -> shrunk comm
  std::map<std::vector<int>, ew_comm*> standby_comms_;  // grown membership -> comm
  std::map<std::vector<int>, int> standby_rounds_;
  std::vector<ew_comm*> retired_;           // parents of splits, freed last
  DpGroupOptions opt_;
  PreparedRecovery* prepared_ = nullptr;
  int events_ = 0;
  std::int64_t snapshot_step_ = -1;
};

// --------------------------------------------------------- in place (D)

// Staged in-place reshard executor (InPlaceSchedule, config D): one buffer
// per rank holds OLD on entry and NEW on exit.  Per phase j each rank gathers
// (staged part into a rotating staging buffer, direct part in place), a
// device-side barrier across the survivors marks "every rank has read phase
// j's OLD bytes", then the staged bytes are flushed.  All gathers and
// flushes are gated on the barrier's error flag, so a timed-out barrier
// vetoes every later write (no OLD byte a lagging peer still needs is lost).
struct InPlaceOptions {
  std::int64_t stage_bytes = 1 << 30;
  std::int64_t phase_bytes = 0;  // 0: 2 * stage_bytes
  int slack = 1;
  int gather_streams = 2;
  int flush_ctas = 64;
  std::int64_t block_bytes = 65536;
  double barrier_timeout_s = 30.0;
};

class InPlaceExecutor {
 public:
  // buf: this rank's single buffer (>= max(OLD, NEW) bytes); replica: the
  // departed member's shard if this rank holds it, else nullptr.  Collective
  // over `ch` (old members; departed members take part in the mapping
  // exchange only when they are still alive — here: all old members call).
  InPlaceExecutor(Channel& ch, const ReshardPlan& rp, void* buf, void* replica,
                  InPlaceOptions opt = {});
  ~InPlaceExecutor();
  InPlaceExecutor(const InPlaceExecutor&) = delete;
  InPlaceExecutor& operator=(const InPlaceExecutor&) = delete;

  // Enqueue every phase on `stream` (+ internal streams joined back);
  // block_sums: device u64 [2 * n_blocks] (caller-zeroed) or nullptr.
  void launch(ew_stream_t stream, std::uint64_t* block_sums);
  bool timed_out() const;
  const InPlaceSchedule& schedule() const { return sched_; }

 private:
  struct Phase;
  ReshardPlan rp_;
  int me_;
  InPlaceOptions opt_;
  InPlaceSchedule sched_;
  void* buf_;
  std::vector<void*> staging_;
  std::vector<std::unique_ptr<Phase>> phases_;
  std::vector<ew_shardmap*> maps_;
  PeerBuffers peers_;
  ew_peer_barrier* barrier_ = nullptr;
  unsigned long long* flags_ = nullptr;
  std::vector<void*> streams_;  // cudaStream_t

  void release();
};

}  // namespace elaskit::b200
