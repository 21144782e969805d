// Multi-process DP recovery in C++ only: one process per rank, no Python.
//
// Each process is one DP rank of an interleaved-ZeRO group (one per GPU, or
// several sharing a GPU: CUDA IPC maps a peer process's allocation on the
// same device too).  Written against the drop-in headers like a reference
// caller of recover_elaswave (sim.cpp:597-722) would be:
//   1. rendezvous on the library's TCP store (rank 0 hosts it);
//   2. steady state: the rank's live shard (synthetic state), its per-step
//      snapshot + checksum rows (kernel (a)), the ring replica of its
//      successor; the DP group (optional NCCL communicator with one prepared
//      shrunk communicator per possible departure) and a PreparedRecovery
//      (every departure planned, lowered, IPC-mapped and bound);
//   3. failure of --drop: the survivors run DpGroup::recover — plan_edit,
//      communicator lookup + first collective, micro-batch reshape, the
//      verified copy, device barrier, conservation over peer memory;
//   4. each survivor checks its NEW bytes against the regenerated target
//      layout and prints its mttr.csv row;
//   5. with --rejoin, the departed process comes back from the free pool
//      (ScaleOut): it builds a joiner-side DpGroup on the same store; in
//      steady state the survivors premap their new shards, everyone
//      prepares the grown communicator (NCCL) and its verified program; the
//      join re-cuts the shards over the grown group; every rank checks its
//      bytes and prints its scale_out mttr.csv row.
//
//   6. with --kill, the departing process is SIGKILLed instead of just
//      leaving: the survivors' heartbeat FailureDetector finds it, and the
//      recovery (no help from the dead process) records the measured
//      detect_s in its mttr.csv row.
//
//   dp_recover --rank R --world N [--port P] [--host H] [--device D]
//              [--scale S] [--drop d] [--nccl] [--rejoin | --kill]
// Exit code 0 iff verified and the bytes match on this rank.
#include <cuda_runtime.h>
#include <signal.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "elaskit/device.hpp"
#include "elaskit/recovery.hpp"

using namespace elaskit;

namespace {

void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
    std::exit(2);
  }
}

struct DeviceBuffer {
  void* p = nullptr;
  explicit DeviceBuffer(std::int64_t bytes) {
    cuda(cudaMalloc(&p, static_cast<std::size_t>(std::max<std::int64_t>(32, (bytes + 31) / 32 * 32))),
         "cudaMalloc");
  }
  ~DeviceBuffer() { cudaFree(p); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

const char* arg(int argc, char** argv, const char* name, const char* dflt) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], name) == 0) return argv[i + 1];
  return dflt;
}

bool flag(int argc, char** argv, const char* name) {
  for (int i = 1; i < argc; ++i)
    if (std::strcmp(argv[i], name) == 0) return true;
  return false;
}

// fill + (optionally) snapshot rows of member r's shard under `layout`
void fill(const PartitionLayout& layout, int r, void* buf, std::uint64_t seed,
          std::uint64_t* rows, void* snap) {
  device::ShardMap m(layout, r);
  device::check(ew_fill_synthetic(m.get(), buf, seed, nullptr));
  if (rows != nullptr) m.snapshot(buf, snap, rows, nullptr);
  cuda(cudaDeviceSynchronize(), "sync");
}

}  // namespace

int main(int argc, char** argv) {
  const int rank = std::atoi(arg(argc, argv, "--rank", "-1"));
  const int world = std::atoi(arg(argc, argv, "--world", "0"));
  const int port = std::atoi(arg(argc, argv, "--port", "29650"));
  const std::string host = arg(argc, argv, "--host", "127.0.0.1");
  const int device_id = std::atoi(arg(argc, argv, "--device", "0"));
  const double scale = std::atof(arg(argc, argv, "--scale", "0.01"));
  const int drop = std::atoi(arg(argc, argv, "--drop", "1"));
  const bool use_nccl = flag(argc, argv, "--nccl");
  const bool rejoin = flag(argc, argv, "--rejoin");
  const bool kill_drop = flag(argc, argv, "--kill");
  if (rank < 0 || world < 2 || rank >= world || drop < 0 || drop >= world ||
      (kill_drop && (drop == 0 || rejoin))) {  // rank 0 hosts the store
    std::fprintf(stderr, "usage: dp_recover --rank R --world N [--drop d] [--nccl] ...\n");
    return 2;
  }
  cuda(cudaSetDevice(device_id), "cudaSetDevice");
  const std::uint64_t seed = 4242;

  // scaled Llama-2 7B ZeRO state (14 B/param), one entry per layer
  std::vector<std::int64_t> layer_bytes;
  layer_bytes.push_back(static_cast<std::int64_t>(131072000 * scale) * 14);
  for (int l = 0; l < 32; ++l) layer_bytes.push_back(static_cast<std::int64_t>(202383360 * scale) * 14);
  layer_bytes.push_back(static_cast<std::int64_t>(131076096 * scale) * 14);
  std::vector<int> members;
  for (int r = 0; r < world; ++r) members.push_back(r);

  try {
    auto store = b200::tcp_store(host, port, rank == 0, 120.0);
    b200::Channel ch(*store, "dp", members, rank);

    // steady state: live shard, snapshot rows, ring replica
    const b200::ReshardPlan whole = b200::ReshardPlan::build(layer_bytes, members, members);
    const int succ = whole.ring.backs_up(rank);
    const std::int64_t n_live = b200::shard_bytes(whole.src, rank);
    const std::int64_t n_rep = b200::shard_bytes(whole.src, succ);
    DeviceBuffer live(n_live), snap(n_live), replica(n_rep), rep_snap(n_rep);
    device::ShardMap live_map(whole.src, rank), rep_map(whole.src, succ);
    DeviceBuffer rows(16 * std::max<std::int64_t>(1, live_map.rows()));
    DeviceBuffer rep_rows(16 * std::max<std::int64_t>(1, rep_map.rows()));
    fill(whole.src, rank, live.p, seed, static_cast<std::uint64_t*>(rows.p), snap.p);
    fill(whole.src, succ, replica.p, seed, static_cast<std::uint64_t*>(rep_rows.p), rep_snap.p);

    ew_comm* comm = nullptr;
    if (use_nccl) {  // one process per GPU: NCCL id through the store
      std::string id(128, '\0');
      if (rank == 0) {
        device::check(ew_comm_unique_id(id.data()));
        store->set("dp/nccl-id", id);
      } else {
        id = store->get("dp/nccl-id");
      }
      device::check(ew_comm_init(id.data(), world, rank, &comm));
    }
    b200::DpGroupOptions gopt;
    gopt.prepare_comms = use_nccl;
    b200::DpGroup group(ch, layer_bytes, comm, gopt);
    b200::PreparedRecovery prepared(ch, layer_bytes, live.p, static_cast<std::uint64_t*>(rows.p),
                                    replica.p, static_cast<std::uint64_t*>(rep_rows.p));
    group.attach(&prepared);
    std::unique_ptr<b200::FailureDetector> detector;
    if (kill_drop)
      detector = std::make_unique<b200::FailureDetector>(ch, "dpr" + std::to_string(port));
    ch.barrier();

    int status = 0;
    double detect_s = 0.0;
    if (kill_drop) {
      if (rank == drop) ::kill(::getpid(), SIGKILL);
      const std::vector<int> dead = detector->wait_for_failure(60.0, &detect_s);
      if (dead != std::vector<int>{drop}) {
        std::fprintf(stderr, "rank %d: detector reported %zu failed members\n", rank, dead.size());
        return 4;
      }
    }
    if (rank != drop) {
      b200::MttrEvent ev = group.recover({drop}, EventKind::FailStop, {}, nullptr, 1);
      ev.detect_s = detect_s;
      // bytes: NEW == the target layout's bytes of the synthetic state
      const b200::ReshardPlan& rp = prepared.plan(drop);
      const std::int64_t n_new = b200::shard_bytes(rp.dst, rank);
      DeviceBuffer expect(n_new);
      fill(rp.dst, rank, expect.p, seed, nullptr, nullptr);
      std::vector<unsigned char> a(static_cast<std::size_t>(n_new)), b(a.size());
      cuda(cudaMemcpy(a.data(), prepared.new_buf(), a.size(), cudaMemcpyDeviceToHost), "D2H");
      cuda(cudaMemcpy(b.data(), expect.p, b.size(), cudaMemcpyDeviceToHost), "D2H");
      const bool bytes_ok = a == b;
      std::printf("rank %d %s verified=%d bytes=%d copy_ms=%.3f comm_repair_ms=%.3f\n", rank,
                  b200::mttr_csv_row(0, ev).c_str(), ev.verified ? 1 : 0, bytes_ok ? 1 : 0,
                  ev.phases.count("copy_s") ? ev.phases.at("copy_s") * 1e3 : -1.0,
                  ev.comm_repair_s * 1e3);
      status = (ev.verified && bytes_ok) ? 0 : 1;
      if (use_nccl) {  // the repaired communicator carries the next step's reduce
        std::int64_t* one = nullptr;
        cuda(cudaMalloc(&one, 8), "cudaMalloc");
        cuda(cudaMemset(one, 0, 8), "memset");
        device::check(ew_allreduce_i64(group.comm(), one, 1, nullptr));
        cuda(cudaDeviceSynchronize(), "sync");
        cudaFree(one);
      }
    }
    if (rejoin) {
      // the departed device returns from the free pool (ScaleOut)
      std::vector<int> survivors;
      for (int m : members)
        if (m != drop) survivors.push_back(m);
      const b200::ReshardPlan back = b200::ReshardPlan::build(layer_bytes, survivors, members);
      const std::int64_t n_back = b200::shard_bytes(back.dst, rank);
      DeviceBuffer grown(n_back);
      std::unique_ptr<b200::DpGroup> joiner;
      b200::DpGroup* g = &group;
      b200::RankBuffers bufs;
      bufs.new_buf = grown.p;
      if (rank == drop) {
        joiner = std::make_unique<b200::DpGroup>(*store, "dp", layer_bytes, survivors, rank, gopt);
        g = joiner.get();
      } else {
        bufs.old_buf = prepared.new_buf();  // the shard recovered above
        g->premap(bufs);                    // steady state after the departure
      }
      g->prepare_join({drop});
      g->prepare_move(EventKind::ScaleOut, {drop}, grown.p);
      const b200::MttrEvent ev = g->recover({drop}, EventKind::ScaleOut, bufs, nullptr, 2);
      DeviceBuffer expect(n_back);
      fill(back.dst, rank, expect.p, seed, nullptr, nullptr);
      std::vector<unsigned char> a(static_cast<std::size_t>(n_back)), b(a.size());
      cuda(cudaMemcpy(a.data(), grown.p, a.size(), cudaMemcpyDeviceToHost), "D2H");
      cuda(cudaMemcpy(b.data(), expect.p, b.size(), cudaMemcpyDeviceToHost), "D2H");
      const bool bytes_ok = a == b;
      const bool grown_ok = g->members() == members;
      std::printf("rank %d rejoin %s verified=%d bytes=%d members=%d prepared=%d copy_ms=%.3f\n",
                  rank, b200::mttr_csv_row(1, ev).c_str(), ev.verified ? 1 : 0, bytes_ok ? 1 : 0,
                  grown_ok ? 1 : 0,
                  ev.phases.count("prepared") ? static_cast<int>(ev.phases.at("prepared")) : -1,
                  ev.phases.count("copy_s") ? ev.phases.at("copy_s") * 1e3 : -1.0);
      if (!(ev.verified && bytes_ok && grown_ok)) status = 1;
      b200::Channel done(*store, "dp-rejoined", members, rank);
      done.barrier();  // the joiner's mappings outlive every peer's reads
    }
    std::fflush(stdout);
    std::vector<int> alive;
    for (int m : members)
      if (!(kill_drop && m == drop)) alive.push_back(m);
    b200::Channel all(*store, "dp-exit", alive, rank);
    all.barrier();  // nobody tears down mappings a peer may still read
    detector.reset();  // stop beating; the segment's owner unlinks it
    if (kill_drop) std::_Exit(status);  // communicators with a dead member: no teardown
    return status;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rank %d: %s\n", rank, e.what());
    return 3;
  }
}
